"""Golden vectors for ingest and the report layer (f3), made
by the REFERENCE in the build container:

    python tests/golden/make_golden_ingest.py

Writes small data files (native MTS and .ts, with comments, missing values,
labels), the reference's parse / finalize / normalize / split outputs for
them, the messages of its ParseErrors on malformed files, and its
emit_report renderings (csv / json / table) of fixed report rows.  Nothing
on the GPU box reads /root/reference.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

from mvdtw import cli, ingest  # noqa: E402

HERE = Path(__file__).resolve().parent
OUT = HERE / "ingest"


def native_text(rng, S, n, D, missing=()):
    lines = ["# synthetic native MTS file", f"{S} {n} {D}"]
    vals = np.cumsum(rng.normal(size=(S, n, D)), axis=1)
    toks = [[repr(float(v)) for v in row] for row in vals.reshape(S * n, D)]
    for (r, k, tok) in missing:
        toks[r][k] = tok
    for r, row in enumerate(toks):
        if r % 17 == 5:
            lines.append("   # interleaved comment")
        if r % 23 == 7:
            lines.append("")
        lines.append(" ".join(row))
    return "\n".join(lines) + "\n"


def ts_text(rng, S, n, D, labels=True):
    lines = ["# sktime subset", "@problemName Synth", "@timeStamps false", "@missing true",
             "@univariate " + ("true" if D == 1 else "false"), f"@dimensions {D}", "@equalLength true",
             f"@seriesLength {n}", "@classLabel " + ("true a b" if labels else "false"), "@data"]
    for s in range(S):
        vals = np.cumsum(rng.normal(size=(D, n)), axis=1)
        segs = [",".join("?" if (s == 1 and k == 0 and t == 3) else repr(float(v)) for t, v in enumerate(vals[k]))
                for k in range(D)]
        if labels:
            segs.append("ab"[s % 2])
        lines.append(":".join(segs))
    return "\n".join(lines) + "\n"


BAD = {
    "bad_header.txt": "3 4\n1 2\n",
    "bad_count.txt": "2 2 2\n1 2\n3 4\n5 6\n",
    "bad_token.txt": "1 2 2\n1 x\n3 4\n",
    "bad_width.txt": "1 2 2\n1 2 3\n3 4\n",
    "bad_empty.txt": "# nothing\n\n",
    "bad_nonpos.txt": "0 2 2\n",
    "bad_ts_directive.ts": "@foo bar\n@data\n1,2:3,4\n",
    "bad_ts_ragged.ts": "@data\n1,2,3:4,5\n",
    "bad_ts_nodata.ts": "@problemName x\n",
    "bad_ts_timestamps.ts": "@timeStamps true\n@data\n1,2\n",
    "bad_ts_before.ts": "1,2:3,4\n@data\n",
}


def main():
    rng = np.random.default_rng(7)
    OUT.mkdir(exist_ok=True)
    files = {
        "native_a.txt": native_text(rng, 12, 20, 3, missing=[(4, 1, "NA"), (30, 0, "?"), (77, 2, "NaN")]),
        "native_b.txt": native_text(rng, 7, 9, 1),
        "ts_a.ts": ts_text(rng, 9, 16, 2, labels=True),
        "ts_b.ts": ts_text(rng, 5, 11, 3, labels=False),
    }
    files.update(BAD)
    for name, text in files.items():
        (OUT / name).write_text(text)
    arrays, meta = {}, {"files": {}, "errors": {}}
    for name in ("native_a.txt", "native_b.txt", "ts_a.ts", "ts_b.ts"):
        path = OUT / name
        raw = ingest.parse_native(path) if name.startswith("native") else ingest.parse_ts_subset(path)
        fin = ingest.finalize(raw)
        nrm = ingest.normalize(raw)
        q, c = ingest.split(nrm, 0.3, 42)
        key = name.split(".")[0]
        arrays[f"{key}_raw"] = raw.values
        arrays[f"{key}_fin"] = fin.values
        arrays[f"{key}_fin_ranges"] = fin.dim_ranges
        arrays[f"{key}_norm"] = nrm.values
        arrays[f"{key}_norm_ranges"] = nrm.dim_ranges
        arrays[f"{key}_q"] = q.values
        arrays[f"{key}_c"] = c.values
        meta["files"][name] = {"name": raw.name, "format": raw.source_format}
    for name in BAD:
        path = OUT / name
        try:
            (ingest.parse_native if name.endswith(".txt") else ingest.parse_ts_subset)(path)
            meta["errors"][name] = None
        except ingest.ParseError as exc:
            meta["errors"][name] = str(exc).replace(str(path), "<path>")
    # report layer: fixed rows, every emitter
    rows = [cli.RunReport("synth", "lb_mv", 10, 3, 12.5, 1.75, None, 700, 100, 0.0123, 0.4567, 0.5, 42,
                          params="lb_mv"),
            cli.RunReport("synth", "tc_dtw", 20, 3, 33.3333333, 2.123456789, 3.5, 400, 200, 0.25, 0.125,
                          0.375, 42, params="tc_dtw(lb_pc) e_ti=0.1 e_pc=0.1 L=2 P=5 K=6 w=6")]
    meta_r = {"host": "box", "threads": 8, "reps": 1, "seed": 42}
    report = {fmt: cli.emit_report(rows, fmt, meta_r) for fmt in ("csv", "json", "table")}
    meta["report"] = report
    meta["report_columns"] = cli.CSV_COLUMNS
    np.savez_compressed(OUT / "ingest.npz", **arrays)
    (OUT / "meta.json").write_text(json.dumps(meta, indent=1))
    print("wrote", sorted(p.name for p in OUT.iterdir()))


if __name__ == "__main__":
    main()
