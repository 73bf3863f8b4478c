"""Edge-case and bit-exactness fixtures for ingest, made by the
REFERENCE in the build container:

    python tests/golden/make_golden_ingest_fuzz.py

* fuzz.json / fuzz.npz: ~100 small native / .ts texts exercising the
  lexical corners the native tokenizer must match (CRLF and lone CR line
  ends, tabs and Unicode spaces, underscores in numbers, inf / nan spellings,
  hex floats, empty tokens, directive case, missing directive arguments,
  labels, comments) with the reference parser's outcome: values + name +
  format, or the exception type and message.
* normalize.json: seeded datasets (D = 1 with a deep pairwise-summation
  tree, D = 2..9 with wide dynamic range so that summation order shows) and
  the reference normalize's mean/std-dependent outputs: dim_ranges, and a
  sha256 of the normalised values' bytes.  The GPU test regenerates the raw
  values from the seed and must reproduce both bit for bit.

Nothing on the GPU box reads /root/reference.
"""

from __future__ import annotations

import hashlib
import json
import sys
import tempfile
from pathlib import Path

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

from mvdtw import ingest  # noqa: E402

OUT = Path(__file__).resolve().parent / "ingest"

NATIVE_CASES = [
    "2 2 1\n1\n2\n3\n4\n",
    "2 2 1\r\n1\r\n2\r\n3\r\n4\r\n",
    "2 2 1\r1\r2\r3\r4\r",
    "2 2 1\n1\n2\n3\n4",
    "  2\t2  2 \n1\t2\n 3  4 \n5\x0b6\n7\x0c8\n",
    "1 2 2\n1\u00a02\n3\u20034\n",
    "1 2 2\n1\x1c2\n3\x1f4\n",
    "1 2 2\n1_000 2.5_5\n1e1_0 .5\n",
    "1 2 2\n1__0 2\n3 4\n",
    "1 2 2\n_1 2\n3 4\n",
    "1 2 2\n1_ 2\n3 4\n",
    "1 2 2\ninf -Infinity\n+nan -NaN\n",
    "1 2 2\nNA na\n? nAn\n",
    "1 2 2\n0x10 2\n3 4\n",
    "1 2 2\n1e 2\n3 4\n",
    "1 2 2\n. 2\n3 4\n",
    "1 2 2\n5. .5\n-0 +0.0\n",
    "1 2 2\n1e400 -1e400\n4.9e-324 2.2250738585072014e-308\n",
    "1 2 2\n0.1 0.2\n0.30000000000000004 123456789012345678901234567890\n",
    "1 2 2\n1 2\n3\n",
    "1 2 2\n1 2\n3 4 5\n",
    "1 2 2\n1 2\n",
    "1 2 2\n1 2\n3 4\n5 6\n",
    "# only\n   # comments\n\n",
    "",
    "\n\n\n",
    "1 2\n",
    "1 2 2 2\n",
    "a 2 2\n",
    "1.0 2 2\n1 2\n3 4\n",
    "+1 2 2\n1 2\n3 4\n",
    "1_0 1 1\n" + "1\n" * 10,
    "0 2 2\n",
    "-1 2 2\n",
    "1 2 2\n\n# mid comment\n1 2\n   \n3 4\n",
    "1 1 3\n1,2 3 4\n",
    "1 1 2\nfoo bar\n",
    "1 1 2\n1 'x'\n",
    "\ufeff1 1 1\n5\n",
    "1 1 1\n\u00e9\n",
    "1 2 1\n 7 \n\t8\t\n",
    "2 1 1\n1\n2\n# trailing comment",
]

TS_HEAD = "@problemName Foo\n@timeStamps false\n@missing true\n@univariate false\n@dimensions 2\n" \
          "@equalLength true\n@seriesLength 3\n@classLabel true a b\n@data\n"
TS_CASES = [
    TS_HEAD + "1,2,3:4,5,6:a\n7,8,9:10,11,12:b\n",
    TS_HEAD.replace("\n", "\r\n") + "1,2,3:4,5,6:a\r\n",
    TS_HEAD + "1, 2 ,3:4,5,6:a\n",
    TS_HEAD + "1,,3:4,5,6:a\n",
    TS_HEAD + "1,?,3:4,NaN,na:a\n",
    TS_HEAD + "1,2,3:4,5,6\n",
    TS_HEAD + "1,2,3:a\n",
    TS_HEAD + "1,2,3:4,5:a\n",
    TS_HEAD + "1,2:4,5:a\n",
    TS_HEAD + "1,2,3:4,5,6:7,8,9:a\n",
    TS_HEAD + "1,2,3:4,5,x:a\n",
    TS_HEAD + "1,2,3:4,5,6:a\n@data\n",
    "@problemname lower\n@data\n1,2:3,4\n5,6:7,8\n",
    "@PROBLEMNAME Upper\n@DATA\n1,2\n",
    "@problemName\n@data\n1,2\n",
    "@problemName a b c\n@data\n1,2\n",
    "@problemName First\n@problemName Second\n@data\n1\n",
    "@timeStamps TRUE\n@data\n1,2\n",
    "@timeStamps\n@data\n1,2\n",
    "@timeStamps false\n@equalLength false\n@data\n1,2\n",
    "@classLabel maybe\n@data\n1,2\n",
    "@classLabel false\n@data\n1,2:3,4\n",
    "@classLabel true x\n@data\n1,2:x\n3,4:y\n",
    "@classLabel true x\n@data\n1,2\n",
    "@dimensions two\n@data\n1,2\n",
    "@dimensions +2\n@data\n1:2\n",
    "@dimensions 1_0\n@data\n1:2\n",
    "@seriesLength 2\n@data\n1,2,3\n",
    "@seriesLength\n@data\n1\n",
    "@targetlabel true\n@data\n1,2\n",
    "@foo bar\n@data\n1\n",
    "@\n@data\n1\n",
    "@data\n",
    "# c\n\n@data\n\n# c\n1,2:3,4\n\n",
    "@data\n1,2:3,4\n1,2,3:4,5,6\n",
    "@data\n1,2:3,4\n1,2:3,4:5,6\n",
    "@data\n1e3,-inf:+inf,1_5\n",
    "@data\n0x1p3,1\n",
    "@data\n1\u00a0,2\n",
    "1,2\n@data\n",
    "@data\r1,2\r3,4\r",
    "@data\n:\n",
    "@data\n1,2:\n",
]


def outcome(fn, text: str, suffix: str):
    with tempfile.TemporaryDirectory() as tmp:
        path = Path(tmp) / f"case{suffix}"
        path.write_text(text, encoding="utf-8", newline="")
        try:
            raw = fn(path)
        except Exception as exc:  # noqa: BLE001 -- the type is part of the fixture
            return {"error": [type(exc).__name__, str(exc).replace(str(path), "<path>")]}, None
        return {"name": raw.name.replace(path.stem, "<stem>"), "format": raw.source_format,
                "shape": list(raw.values.shape)}, raw.values


def fuzz():
    cases, arrays = [], {}
    for i, text in enumerate(NATIVE_CASES):
        rec, vals = outcome(ingest.parse_native, text, ".txt")
        cases.append({"fmt": "native", "text": text, **rec})
        if vals is not None:
            arrays[f"c{len(cases) - 1}"] = vals
    for i, text in enumerate(TS_CASES):
        rec, vals = outcome(ingest.parse_ts_subset, text, ".ts")
        cases.append({"fmt": "ts", "text": text, **rec})
        if vals is not None:
            arrays[f"c{len(cases) - 1}"] = vals
    (OUT / "fuzz.json").write_text(json.dumps(cases, indent=1, ensure_ascii=True))
    np.savez_compressed(OUT / "fuzz.npz", **arrays)
    return len(cases)


# (seed, S, n, D, scale spread): raw = normal * 10**uniform(-spread, spread) + offset
NORM_CASES = [(1, 300, 700, 1, 6), (2, 40, 50, 1, 3), (3, 1, 5, 1, 2), (4, 1, 200, 1, 8), (5, 500, 100, 2, 6),
              (6, 200, 300, 3, 8), (7, 64, 129, 5, 4), (8, 30, 1000, 7, 6), (9, 10, 17, 9, 2), (10, 3, 1, 4, 1)]


def normal_raw(seed, S, n, D, spread):
    """The raw values of one normalize fixture (the GPU test calls this same
    recipe, copied into tests/test_gpu_ingest.py)."""
    rng = np.random.default_rng(seed)
    v = rng.normal(size=(S, n, D)) * 10.0 ** rng.uniform(-spread, spread, size=(S, n, D)) + rng.normal(size=D) * 50
    v[rng.random(size=v.shape) < 0.01] = np.nan
    if D > 2:
        v[:, :, 1] = 3.25  # a zero-variance dimension
    return v


def normalize_cases():
    recs = []
    for seed, S, n, D, spread in NORM_CASES:
        raw = ingest.RawDataset("x", normal_raw(seed, S, n, D, spread), "native")
        ds = ingest.normalize(raw)
        recs.append({"seed": seed, "S": S, "n": n, "D": D, "spread": spread,
                     "dim_ranges": [float(x).hex() for x in ds.dim_ranges],
                     "sha256": hashlib.sha256(np.ascontiguousarray(ds.values).tobytes()).hexdigest()})
    (OUT / "normalize.json").write_text(json.dumps(recs, indent=1))
    return len(recs)


if __name__ == "__main__":
    print("fuzz cases:", fuzz(), " normalize cases:", normalize_cases())
