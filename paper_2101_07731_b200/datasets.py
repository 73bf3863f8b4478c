"""Seeded synthetic workloads for the BASELINE.json configs C0-C4.

The paper measures on the UCR multivariate archive, which is not available
here; these generators stand in for it with the shapes, sizes and value
distributions BASELINE.json names.  Rows [0, N_c)
are candidates and rows [N_c, N_c + N_q) are queries.  Values are
z-normalised per dimension over the whole drawn set, as the reference's
``normalize`` does (ingest.py:245-261); fp32 configs are cast after
normalising, and the per-dimension ``dim_range`` (ingest.py:234-236) is
measured on the values actually searched.

Generators:
  random walk (C0, C1, C3): cumsum of N(0, 1) steps along time, the
      construction of synth.random_walk_dataset (synth.py:24-31); C1 adds
      N(0, 0.1) noise.
  sinusoid mixture (C2, C4): no reference generator exists; the
      recipe pinned here is: per (prototype, dim) frequency f ~ U[1, 8]
      cycles and phase phi ~ U[0, 2pi); class uniform per series; linear
      time warp t' = t (1 + a), a ~ U[-0.1, 0.1]; value
      sin(2 pi f t' / L + phi) + N(0, 0.2).

This is host-side input generation, not the search path.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class ConfigSpec:
    name: str
    n_candidates: int
    n_queries: int
    length: int
    dims: int
    dtype: str  # "f64" | "f32"
    window_fracs: tuple
    family: str  # "walk" | "walk_noise" | "sines"
    prototypes: int = 0

    def windows(self) -> list[int]:
        # W = int(frac * L)  (SURVEY ledger D4)
        return [int(f * self.length) for f in self.window_fracs]


CONFIGS = {
    "C0": ConfigSpec("C0", 200, 20, 128, 3, "f64", (0.10,), "walk"),
    "C1": ConfigSpec("C1", 5000, 500, 256, 5, "f32", (0.05, 0.20), "walk_noise"),
    "C2": ConfigSpec("C2", 50000, 1000, 64, 20, "f32", (0.10,), "sines", 10),
    "C3": ConfigSpec("C3", 2000, 100, 1024, 8, "f64", (0.10,), "walk"),
    "C4": ConfigSpec("C4", 1000000, 10000, 128, 6, "f32", (0.10,), "sines", 50),
}


@dataclass
class Workload:
    spec: ConfigSpec
    candidates: np.ndarray  # (N_c, L, d), float64 or float32
    queries: np.ndarray  # (N_q, L, d)
    dim_range: np.ndarray  # (d,) float64
    seed: int

    @property
    def dtype(self) -> str:
        return self.spec.dtype


def _normalize_exact(vals: np.ndarray) -> np.ndarray:
    """Restates ingest.normalize (ingest.py:253-261) on a float64 array."""
    flat = vals.reshape(-1, vals.shape[2])
    mean = flat.mean(axis=0)
    std = flat.std(axis=0)
    safe = np.where(std > 0.0, std, 1.0)
    normed = (vals - mean) / safe
    normed[..., std == 0.0] = 0.0
    return normed


def _ranges(vals: np.ndarray) -> np.ndarray:
    flat = vals.reshape(-1, vals.shape[2])
    return (flat.max(axis=0).astype(np.float64) - flat.min(axis=0).astype(np.float64))


def _walk(spec: ConfigSpec, S: int, rng: np.random.Generator) -> np.ndarray:
    vals = np.cumsum(rng.normal(0.0, 1.0, (S, spec.length, spec.dims)), axis=1)
    if spec.family == "walk_noise":
        vals = vals + rng.normal(0.0, 0.1, vals.shape)
    return vals


def _sines_chunked(spec: ConfigSpec, S: int, rng: np.random.Generator, chunk: int = 65536) -> np.ndarray:
    """Sinusoid mixture in float32 chunks (C4 is 7.7e8 values); returns the
    normalised float32 array.  Statistics accumulate in float64."""
    L, d, P = spec.length, spec.dims, spec.prototypes
    freq = rng.uniform(1.0, 8.0, (P, d))
    phase = rng.uniform(0.0, 2.0 * np.pi, (P, d))
    classes = rng.integers(0, P, S)
    warp = rng.uniform(-0.1, 0.1, S)
    t = np.arange(L, dtype=np.float64)
    out = np.empty((S, L, d), dtype=np.float32)
    two_pi_over_L = 2.0 * np.pi / L
    for s0 in range(0, S, chunk):
        s1 = min(S, s0 + chunk)
        tw = t[None, :] * (1.0 + warp[s0:s1, None])  # (c, L)
        arg = (freq[classes[s0:s1]][:, None, :] * tw[:, :, None]) * two_pi_over_L \
            + phase[classes[s0:s1]][:, None, :]
        v = np.sin(arg.astype(np.float32))
        v += rng.standard_normal((s1 - s0, L, d), dtype=np.float32) * np.float32(0.2)
        out[s0:s1] = v
    # two-pass per-dimension z-normalisation over the whole set
    flat = out.reshape(-1, d)
    n_rows = flat.shape[0]
    step = 1 << 22
    s = np.zeros(d)
    for r0 in range(0, n_rows, step):
        s += flat[r0:r0 + step].sum(axis=0, dtype=np.float64)
    mean = s / n_rows
    ss = np.zeros(d)
    for r0 in range(0, n_rows, step):
        x = flat[r0:r0 + step].astype(np.float64) - mean
        ss += (x * x).sum(axis=0)
    std = np.sqrt(ss / n_rows)
    safe = np.where(std > 0.0, std, 1.0)
    for r0 in range(0, n_rows, step):
        x = (flat[r0:r0 + step].astype(np.float64) - mean) / safe
        x[:, std == 0.0] = 0.0
        flat[r0:r0 + step] = x.astype(np.float32)
    return out


def make_workload(name: str, seed: int = 0, n_candidates: int | None = None,
                  n_queries: int | None = None) -> Workload:
    """Generate config `name` (C0..C4).  Overriding the counts keeps the
    recipe (used for reduced-size parity cases); the full draw is
    N_c + N_q series in that order."""
    spec = CONFIGS[name]
    n_c = spec.n_candidates if n_candidates is None else int(n_candidates)
    n_q = spec.n_queries if n_queries is None else int(n_queries)
    S = n_c + n_q
    rng = np.random.default_rng(seed)
    if spec.family in ("walk", "walk_noise"):
        vals = _normalize_exact(_walk(spec, S, rng))
        if spec.dtype == "f32":
            vals = vals.astype(np.float32)
    else:
        vals = _sines_chunked(spec, S, rng)
        if spec.dtype == "f64":
            vals = vals.astype(np.float64)
    vals = np.ascontiguousarray(vals)
    return Workload(spec, vals[:n_c], vals[n_c:], _ranges(vals), seed)
