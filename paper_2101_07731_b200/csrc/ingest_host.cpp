// Host-side dataset tokenizers: the reference's two text
// formats (mvdtw ingest.py:92-126 native MTS, ingest.py:157-231 the sktime
// .ts subset) parsed in one pass over the file bytes straight into the
// caller's (pinned) float64 buffer.  The Python layer (ingest.py) owns file
// reading and turns the error record below into the reference's ParseError
// messages; this file only scans and converts.
//
// Lexical rules are Python's, because the reference tokenizes with str
// methods and converts with float()/int():
//   * lines end at "\n", "\r\n" or "\r" (text-mode universal newlines);
//   * whitespace is every code point str.isspace() accepts (ASCII and the
//     UTF-8 encoded Unicode separators), for strip() and split();
//   * a number follows float()'s grammar: optional sign, digits with single
//     underscores between them, optional fraction and exponent, or
//     inf / infinity / nan in any case.  Hex floats and C-only forms are
//     rejected.  Conversion is glibc strtod (correctly rounded, like
//     CPython's dtoa), so values are bit-identical.
//   * Non-ASCII digits, which float() would accept, are rejected here.
#include <cerrno>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "tcdtw.h"

namespace {

using Info = tcdtw_parse_info;

// ------------------------------------------------------------- characters
// Byte length of the str.isspace() code point starting at p (0 if none).
inline int space_len(const unsigned char* p, const unsigned char* end) {
    const unsigned char b = p[0];
    if (b == ' ' || (b >= 0x09 && b <= 0x0d) || (b >= 0x1c && b <= 0x1f)) return 1;
    if (b < 0x80) return 0;
    const ptrdiff_t left = end - p;
    if (b == 0xc2 && left >= 2 && (p[1] == 0x85 || p[1] == 0xa0)) return 2;  // U+0085, U+00A0
    if (left < 3) return 0;
    const unsigned c1 = p[1], c2 = p[2];
    if (b == 0xe1 && c1 == 0x9a && c2 == 0x80) return 3;                       // U+1680
    if (b == 0xe2 && c1 == 0x80 && ((c2 >= 0x80 && c2 <= 0x8a) || c2 == 0xa8 || c2 == 0xa9 || c2 == 0xaf))
        return 3;                                                              // U+2000-200A, 2028, 2029, 202F
    if (b == 0xe2 && c1 == 0x81 && c2 == 0x9f) return 3;                       // U+205F
    if (b == 0xe3 && c1 == 0x80 && c2 == 0x80) return 3;                       // U+3000
    return 0;
}

struct Span {
    const unsigned char* b;
    const unsigned char* e;
    bool empty() const { return b == e; }
    size_t size() const { return (size_t)(e - b); }
};

// str.strip()
Span strip(Span s) {
    while (s.b < s.e) {
        const int k = space_len(s.b, s.e);
        if (!k) break;
        s.b += k;
    }
    // trailing: walk forward to find the last non-space code point end
    const unsigned char* last = s.b;
    for (const unsigned char* p = s.b; p < s.e;) {
        const int k = space_len(p, s.e);
        if (k) {
            p += k;
        } else {
            ++p;
            while (p < s.e && (*p & 0xc0) == 0x80) ++p;  // rest of a UTF-8 sequence
            last = p;
        }
    }
    s.e = last;
    return s;
}

// Next str.split() field of s starting at *pos; false when none is left.
bool next_field(Span s, const unsigned char** pos, Span* out) {
    const unsigned char* p = *pos;
    while (p < s.e) {
        const int k = space_len(p, s.e);
        if (!k) break;
        p += k;
    }
    if (p >= s.e) {
        *pos = p;
        return false;
    }
    const unsigned char* start = p;
    while (p < s.e && !space_len(p, s.e)) {
        ++p;
        while (p < s.e && (*p & 0xc0) == 0x80) ++p;
    }
    *out = Span{start, p};
    *pos = p;
    return true;
}

// Line iterator with universal newlines; numbers lines from 1.
struct Lines {
    const unsigned char* p;
    const unsigned char* end;
    int64_t no = 0;
    bool done = false;
    bool next(Span* line) {
        if (done) return false;
        const unsigned char* s = p;
        while (p < end && *p != '\n' && *p != '\r') ++p;
        *line = Span{s, p};
        ++no;
        if (p >= end) {
            done = true;  // the text after the last break is a (possibly empty) last line
            return true;
        }
        if (*p == '\r' && p + 1 < end && p[1] == '\n') ++p;
        ++p;
        return true;
    }
};

inline char lower(unsigned char c) { return (c >= 'A' && c <= 'Z') ? (char)(c + 32) : (char)c; }

bool equals_ci(Span s, const char* word) {
    const size_t n = strlen(word);
    if (s.size() != n) return false;
    for (size_t i = 0; i < n; ++i)
        if (lower(s.b[i]) != word[i]) return false;
    return true;
}

bool equals(Span s, const char* word) { return s.size() == strlen(word) && memcmp(s.b, word, s.size()) == 0; }

// digits with single underscores between digits; appends the digits to buf
bool digit_run(const unsigned char*& p, const unsigned char* e, std::string& buf) {
    if (p >= e || *p < '0' || *p > '9') return false;
    while (p < e) {
        if (*p >= '0' && *p <= '9') {
            buf.push_back((char)*p++);
        } else if (*p == '_' && p + 1 < e && p[1] >= '0' && p[1] <= '9') {
            ++p;
        } else {
            break;
        }
    }
    return true;
}

// float() of one stripped token; false = not a number
bool to_double(Span t, double* out, std::string& buf) {
    const unsigned char* p = t.b;
    const unsigned char* e = t.e;
    buf.clear();
    if (p < e && (*p == '+' || *p == '-')) buf.push_back((char)*p++);
    const Span rest{p, e};
    if (equals_ci(rest, "inf") || equals_ci(rest, "infinity")) {
        *out = (!buf.empty() && buf[0] == '-') ? -INFINITY : INFINITY;
        return true;
    }
    if (equals_ci(rest, "nan")) {
        *out = (!buf.empty() && buf[0] == '-') ? -NAN : NAN;
        return true;
    }
    const bool int_part = digit_run(p, e, buf);
    bool frac_part = false;
    if (p < e && *p == '.') {
        buf.push_back('.');
        ++p;
        frac_part = digit_run(p, e, buf);
    }
    if (!int_part && !frac_part) return false;
    if (p < e && (*p == 'e' || *p == 'E')) {
        buf.push_back('e');
        ++p;
        if (p < e && (*p == '+' || *p == '-')) buf.push_back((char)*p++);
        if (!digit_run(p, e, buf)) return false;
    }
    if (p != e) return false;
    errno = 0;
    *out = strtod(buf.c_str(), nullptr);  // overflow gives +-inf, as float() does
    return true;
}

// int() of one stripped token (ASCII digits, underscores, sign); saturates
bool to_int(Span t, int64_t* out) {
    const unsigned char* p = t.b;
    const unsigned char* e = t.e;
    bool neg = false;
    if (p < e && (*p == '+' || *p == '-')) neg = *p++ == '-';
    std::string digits;
    if (!digit_run(p, e, digits) || p != e) return false;
    int64_t v = 0;
    for (char c : digits) {
        if (v > (INT64_MAX - 9) / 10) {
            v = INT64_MAX;
            break;
        }
        v = v * 10 + (c - '0');
    }
    *out = neg ? -v : v;
    return true;
}

int fail(Info* info, int code, int64_t line, Span tok, const unsigned char* base) {
    info->error = code;
    info->line = line;
    info->tok_off = tok.b ? (int64_t)(tok.b - base) : -1;
    info->tok_len = tok.b ? (int64_t)tok.size() : 0;
    return TCDTW_INVALID_INPUT;
}

bool is_missing(Span t) { return equals_ci(t, "na") || equals_ci(t, "nan") || equals(t, "?"); }

// ----------------------------------------------------------- native format
int parse_native(const unsigned char* text, size_t len, double* values, int64_t cap, Info* info) {
    Lines lines{text, text + len};
    Span line{};
    std::string buf;
    // header: the first line that is neither blank nor a comment
    bool have_header = false;
    while (lines.next(&line)) {
        const Span s = strip(line);
        if (s.empty() || s.b[0] == '#') continue;
        have_header = true;
        const unsigned char* pos = s.b;
        Span f[4];
        int nf = 0;
        while (nf < 4 && next_field(s, &pos, &f[nf])) ++nf;
        if (nf != 3) return fail(info, TCDTW_PARSE_HEADER_FIELDS, lines.no, Span{}, text);
        int64_t v[3];
        for (int k = 0; k < 3; ++k)
            if (!to_int(f[k], &v[k])) return fail(info, TCDTW_PARSE_HEADER_INT, lines.no, f[k], text);
        if (v[0] < 1 || v[1] < 1 || v[2] < 1) return fail(info, TCDTW_PARSE_HEADER_POSITIVE, lines.no, Span{}, text);
        info->num_series = v[0];
        info->length = v[1];
        info->dims = v[2];
        info->line = lines.no;
        break;
    }
    if (!have_header) return fail(info, TCDTW_PARSE_EMPTY, 0, Span{}, text);
    const int64_t S = info->num_series, n = info->length, D = info->dims;
    const int64_t want = (S > INT64_MAX / n) ? INT64_MAX : S * n;
    // the reference counts the value lines before reading any of them
    const Lines body = lines;
    int64_t rows = 0;
    while (lines.next(&line)) {
        const Span s = strip(line);
        if (!s.empty() && s.b[0] != '#') ++rows;
    }
    info->expected = want;
    info->found = rows;
    if (rows != want) return fail(info, TCDTW_PARSE_LINE_COUNT, 0, Span{}, text);
    if (values == nullptr) return TCDTW_OK;  // shape query
    if (D > 0 && cap / D < rows) return TCDTW_WORKSPACE_TOO_SMALL;
    lines = body;
    double* out = values;
    while (lines.next(&line)) {
        const Span s = strip(line);
        if (s.empty() || s.b[0] == '#') continue;
        // count first (the reference checks the width before converting)
        const unsigned char* pos = s.b;
        Span f{};
        int64_t k = 0;
        while (next_field(s, &pos, &f)) ++k;
        if (k != D) {
            info->expected = D;
            info->found = k;
            return fail(info, TCDTW_PARSE_ROW_WIDTH, lines.no, Span{}, text);
        }
        pos = s.b;
        while (next_field(s, &pos, &f)) {
            if (is_missing(f)) {
                *out++ = NAN;
            } else if (!to_double(f, out++, buf)) {
                return fail(info, TCDTW_PARSE_TOKEN, lines.no, f, text);
            }
        }
    }
    return TCDTW_OK;
}

// ------------------------------------------------------------ .ts subset
enum Directive { D_UNKNOWN, D_PROBLEMNAME, D_TIMESTAMPS, D_MISSING, D_UNIVARIATE, D_DIMENSION, D_EQUALLENGTH,
                 D_SERIESLENGTH, D_CLASSLABEL, D_TARGETLABEL, D_DATA };

Directive directive_of(Span key) {
    static const struct {
        const char* word;
        Directive d;
    } table[] = {{"problemname", D_PROBLEMNAME}, {"timestamps", D_TIMESTAMPS},   {"missing", D_MISSING},
                 {"univariate", D_UNIVARIATE},   {"dimension", D_DIMENSION},     {"dimensions", D_DIMENSION},
                 {"equallength", D_EQUALLENGTH}, {"serieslength", D_SERIESLENGTH}, {"classlabel", D_CLASSLABEL},
                 {"targetlabel", D_TARGETLABEL}, {"data", D_DATA}};
    for (const auto& t : table)
        if (equals_ci(key, t.word)) return t.d;
    return D_UNKNOWN;
}

// the .ts boolean arguments are exactly "true" / "false"
int ts_flag(Span arg, bool* v) {
    if (equals(arg, "true")) {
        *v = true;
        return 0;
    }
    if (equals(arg, "false")) {
        *v = false;
        return 0;
    }
    return 1;
}

// Comma-separated tokens of one ':' segment, each stripped, in order.
template <typename F>
void for_each_token(Span seg, F&& f) {
    const unsigned char* p = seg.b;
    while (true) {
        const unsigned char* q = p;
        while (q < seg.e && *q != ',') ++q;
        if (!f(strip(Span{p, q}))) return;
        if (q >= seg.e) return;
        p = q + 1;
    }
}

int parse_ts(const unsigned char* text, size_t len, double* values, int64_t cap, Info* info) {
    Lines lines{text, text + len};
    Span line{};
    std::string buf;
    std::vector<double> cols;  // one series, [dim][t]
    int64_t dims_decl = 0, len_decl = 0, n_series = 0, shape_n = -1, shape_d = -1;
    bool has_dims = false, has_len = false, labelled = false, in_data = false;
    while (lines.next(&line)) {
        const Span s = strip(line);
        if (s.empty() || s.b[0] == '#') continue;
        if (s.b[0] == '@') {
            if (in_data) return fail(info, TCDTW_PARSE_TS_AFTER_DATA, lines.no, Span{}, text);
            const Span body{s.b + 1, s.e};
            const unsigned char* pos = body.b;
            Span key{}, arg{};
            const bool has_key = next_field(body, &pos, &key);
            const bool has_arg = has_key && next_field(body, &pos, &arg);
            const Directive dv = has_key ? directive_of(key) : D_UNKNOWN;
            if (dv == D_UNKNOWN) return fail(info, TCDTW_PARSE_TS_DIRECTIVE, lines.no, has_key ? key : Span{}, text);
            bool flag = false;
            switch (dv) {
                case D_DATA:
                    in_data = true;
                    break;
                case D_TIMESTAMPS:
                    if (!has_arg || ts_flag(arg, &flag)) return fail(info, TCDTW_PARSE_TS_FLAG, lines.no, arg, text);
                    if (flag) return fail(info, TCDTW_PARSE_TS_TIMESTAMPS, lines.no, Span{}, text);
                    break;
                case D_EQUALLENGTH:
                    if (!has_arg || ts_flag(arg, &flag)) return fail(info, TCDTW_PARSE_TS_FLAG, lines.no, arg, text);
                    if (!flag) return fail(info, TCDTW_PARSE_TS_UNEQUAL, lines.no, Span{}, text);
                    break;
                case D_DIMENSION:
                case D_SERIESLENGTH: {
                    int64_t v = 0;
                    if (!has_arg || !to_int(arg, &v)) return fail(info, TCDTW_PARSE_TS_INT_ARG, lines.no, arg, text);
                    if (dv == D_DIMENSION) {
                        dims_decl = v;
                        has_dims = true;
                    } else {
                        len_decl = v;
                        has_len = true;
                    }
                    break;
                }
                case D_CLASSLABEL:
                    if (!has_arg || ts_flag(arg, &labelled)) return fail(info, TCDTW_PARSE_TS_FLAG, lines.no, arg, text);
                    break;
                case D_PROBLEMNAME:
                    if (has_arg) {
                        info->name_off = (int64_t)(arg.b - text);
                        info->name_len = (int64_t)arg.size();
                    }
                    break;
                default:
                    break;
            }
            continue;
        }
        if (!in_data) return fail(info, TCDTW_PARSE_TS_BEFORE_DATA, lines.no, Span{}, text);
        // ':' segments = dimensions; with class labels the last one is the label
        int64_t nseg = 1;
        for (const unsigned char* p = s.b; p < s.e; ++p) nseg += (*p == ':');
        if (labelled) {
            if (nseg < 2) return fail(info, TCDTW_PARSE_TS_LABEL, lines.no, Span{}, text);
            --nseg;
        }
        if (has_dims && nseg != dims_decl) {
            info->expected = dims_decl;
            info->found = nseg;
            return fail(info, TCDTW_PARSE_TS_DIMS, lines.no, Span{}, text);
        }
        // every token is converted (segment order) before the shape checks
        cols.clear();
        int64_t n0 = -1;
        bool ragged = false;
        const unsigned char* p = s.b;
        for (int64_t k = 0; k < nseg; ++k) {
            const unsigned char* q = p;
            while (q < s.e && *q != ':') ++q;
            int64_t t = 0;
            Span bad{};
            bool ok = true;
            for_each_token(Span{p, q}, [&](Span tok) {
                double v = NAN;
                if (!is_missing(tok) && !to_double(tok, &v, buf)) {
                    bad = tok;
                    ok = false;
                    return false;
                }
                cols.push_back(v);
                ++t;
                return true;
            });
            if (!ok) return fail(info, TCDTW_PARSE_TOKEN, lines.no, bad, text);
            if (n0 < 0) n0 = t;
            ragged |= (t != n0);
            p = q + 1;
        }
        if (ragged) return fail(info, TCDTW_PARSE_TS_RAGGED, lines.no, Span{}, text);
        if (has_len && n0 != len_decl) {
            info->expected = len_decl;
            info->found = n0;
            return fail(info, TCDTW_PARSE_TS_LENGTH, lines.no, Span{}, text);
        }
        if (shape_n < 0) {
            shape_n = n0;
            shape_d = nseg;
        } else if (n0 != shape_n || nseg != shape_d) {
            return fail(info, TCDTW_PARSE_TS_SHAPE, lines.no, Span{}, text);
        }
        if (values != nullptr) {  // (length, dims) = transpose of the segments
            const int64_t per = shape_n * shape_d;
            if (per > 0 && cap / per <= n_series) return TCDTW_WORKSPACE_TOO_SMALL;
            double* dst = values + n_series * per;
            for (int64_t k = 0; k < shape_d; ++k)
                for (int64_t t = 0; t < shape_n; ++t) dst[t * shape_d + k] = cols[k * shape_n + t];
        }
        ++n_series;
    }
    if (n_series == 0) return fail(info, TCDTW_PARSE_TS_NO_DATA, 0, Span{}, text);
    info->num_series = n_series;
    info->length = shape_n;
    info->dims = shape_d;
    return TCDTW_OK;
}

}  // namespace

extern "C" {

int tcdtw_parse_text(int32_t format, const char* text, size_t len, double* values, int64_t capacity,
                     tcdtw_parse_info* info) {
    if (info == nullptr || (text == nullptr && len > 0)) return TCDTW_INVALID_INPUT;
    memset(info, 0, sizeof(*info));
    info->tok_off = -1;
    info->name_off = -1;
    const unsigned char* t = reinterpret_cast<const unsigned char*>(text ? text : "");
    if (format == TCDTW_FORMAT_NATIVE) return parse_native(t, len, values, capacity, info);
    if (format == TCDTW_FORMAT_TS) return parse_ts(t, len, values, capacity, info);
    return TCDTW_INVALID_INPUT;
}

}  // extern "C"
