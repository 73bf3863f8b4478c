#!/usr/bin/env python
"""Benchmark: batched windowed-DTW 1-NN search (TC-DTW cascade) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C4] [--impl ours|reference]

A step is one pass of the hot path over one batch of synthetic input: every
query of the config searched against the whole (sharded) candidate
collection, which stays resident in HBM like a database index (it is 3 GB
at C4, far above the 126 MB L2, so no L2 flush is needed between steps).

value  = whole-job queries/s, device-timed (CUDA events), queries resident.
e2e    = queries/s through the public API (SearchIndex.search) with pinned
         host query buffers: H2D of the queries and D2H of (index, distance)
         inside the timed region.
Rank 0 prints one JSON line.  With --impl reference the CPU arm (the C port
of the reference algorithm in oracle/, all host threads) runs instead.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "1-NN queries/sec (GCUPS and roofline reported alongside)"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C4")
    ap.add_argument("--window-index", type=int, default=0)
    ap.add_argument("--method", default="lb_mv", help="a Method value, or auto (GPU-cost choice, SURVEY 8f f1)")
    ap.add_argument("--queries", type=int, default=0, help="use only the first Q queries (0 = all)")
    ap.add_argument("--candidates", type=int, default=0, help="override N_c (0 = config)")
    ap.add_argument("--batch", type=int, default=0)
    ap.add_argument("--seeds", type=int, default=0)
    ap.add_argument("--cpu-seconds", type=float, default=15.0, help="CPU baseline sample budget")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-exchange", action="store_true", help="skip the d_best all-reduce between phases")
    ap.add_argument("--dist-backend", default="nccl", help="nccl (one GPU per rank) or gloo (testing)")
    ap.add_argument("--no-cascade", action="store_true", help="A/B: DTW abandons on row minima only")
    ap.add_argument("--reverse-pc", action="store_true",
                    help="f2: with an LB_PC second stage, also prune on the reverse LB_PC (candidate box sets)")
    ap.add_argument("--reverse-bound", action="store_true",
                    help="also prune on LB_MV(q, env(c)) from the candidate-side index (SURVEY 8f f2)")
    return ap.parse_args()


# ------------------------------------------------------------------ helpers
def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


class ClockSampler:
    """SM clocks and throttle reasons sampled DURING the timed region: NVML
    (nvidia-ml-py) polled every 5 ms from a thread, plus one sample at entry
    and exit, so even millisecond-long regions get samples; nvidia-smi
    (-lms 100) if NVML is unavailable."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4}

    def __init__(self, gpu_index: int, period_s: float = 0.005):
        self.gpu = gpu_index
        self.period = period_s
        self.rows = []  # (sm_mhz, max_mhz, reason bits)
        self._stop = None
        self._thread = None
        self._nvml = None
        self._h = None

    def _sample(self):
        n = self._nvml
        reasons = getattr(n, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
            n.nvmlDeviceGetCurrentClocksThrottleReasons
        self.rows.append((n.nvmlDeviceGetClockInfo(self._h, n.NVML_CLOCK_SM),
                          n.nvmlDeviceGetMaxClockInfo(self._h, n.NVML_CLOCK_SM), int(reasons(self._h))))

    def _loop(self):
        while not self._stop.wait(self.period):
            try:
                self._sample()
            except Exception:
                return

    def __enter__(self):
        import threading

        try:
            import pynvml

            pynvml.nvmlInit()
            self._nvml = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(self._physical_index())
            self._sample()
        except Exception:
            self._nvml = None
            return self
        self._stop = threading.Event()
        self._thread = threading.Thread(target=self._loop, daemon=True)
        self._thread.start()
        return self

    def _physical_index(self) -> int:
        vis = os.environ.get("CUDA_VISIBLE_DEVICES")
        if vis:
            ids = [v.strip() for v in vis.split(",") if v.strip()]
            if self.gpu < len(ids) and ids[self.gpu].isdigit():
                return int(ids[self.gpu])
        return self.gpu

    def __exit__(self, *a):
        if self._thread is not None:
            self._stop.set()
            self._thread.join(timeout=2)
        if self._nvml is not None:
            try:
                self._sample()
            except Exception:
                pass

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        reasons = sorted(nm for nm, bit in self.REASONS.items() if any(r[2] & bit for r in self.rows))
        return {"sm_mhz": statistics.median(r[0] for r in self.rows), "sm_max_mhz": max(r[1] for r in self.rows),
                "reasons": reasons, "samples": len(self.rows), "source": "nvml"}


def traffic_from_profile(cells_per_launch=None):
    """DRAM bytes (read + write) per launch of the dominant kernel, from the
    committed ncu --set full capture (profiles/dtw_lane_traffic.json, taken
    on a reduced C4 run) scaled by DP cells per launch; None if absent."""
    p = ROOT / "profiles" / "dtw_lane_traffic.json"
    if p.exists() and cells_per_launch:
        try:
            j = json.loads(p.read_text())
            return j["dram_bytes"] / j["dtw_cells"] * cells_per_launch
        except Exception:
            pass
    return None


def measured_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            return json.loads(p.read_text())
        except Exception:
            pass
    return {}


def index_envelope_stats(index, w, _lib, reps=5):
    """The candidate-side index build: envelopes of the whole
    shard by the streaming envelope kernel, timed with CUDA events on the
    launching stream.  HBM-bound: reads n*d and writes 2*n*d elements per
    series (3*N*L*d*s bytes)."""
    import torch

    N, n, d = index.candidates.shape
    es = index.candidates.element_size()
    up = torch.empty_like(index.candidates)
    lo = torch.empty_like(index.candidates)
    code = _lib.dtype_code(index.dtype)
    L = _lib.lib()
    weff = min(int(w), n - 1)

    def go():
        _lib.check(L.tcdtw_build_envelope(code, index.candidates.data_ptr(), N, n, d, weff, up.data_ptr(),
                                          lo.data_ptr(), _lib.stream_ptr()), "build_envelope")

    go()
    torch.cuda.synchronize()
    ms = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        go()
        e1.record()
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    t = statistics.median(ms)
    nbytes = 3 * N * n * d * es
    peak = measured_peaks().get("hbm_gbs")
    gbs = nbytes / (t / 1e3) / 1e9
    del up, lo
    return {"kernel": "envelope_vh_kernel (TMA bulk loads, van Herk in registers; k <= 32)", "bound": "hbm", "series": int(N), "ms": t,
            "algorithmic_bytes": nbytes, "achieved": gbs, "peak": peak, "unit": "GB/s",
            "frac": gbs / peak if peak else None,
            "peak_source": "MEASURED_PEAKS.json hbm_gbs (driver copy test)"}


# -------------------------------------------------------- CPU (oracle) legs
def host_cpu() -> str:
    """The host CPU model (lscpu's "Model name", from /proc/cpuinfo)."""
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.lower().startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform

    return platform.processor() or "unknown"


def cpu_queries_per_sec(wl, w, method, advanced, n_queries_hint, budget_s, threads=0, knobs=None):
    """Time the C port of the reference algorithm (oracle/, all threads) on
    a bounded sample of the queries against the full collection."""
    from oracle import oracle as O

    cands64 = wl.candidates.astype(np.float64)
    params = O.make_params(w, method, **(knobs or {}))
    threads = threads or (os.cpu_count() or 1)
    # one probe query on one thread to size the sample
    t0 = time.perf_counter()
    O.nn_search_batch(wl.queries[:1].astype(np.float64), cands64, params, advanced, wl.dim_range, n_threads=1)
    t1 = time.perf_counter() - t0
    per_query = max(t1, 1e-3)
    nq = int(max(1, min(len(wl.queries), n_queries_hint or 10 ** 9,
                        round(budget_s / per_query * max(1, threads) * 0.8))))
    nq = max(nq, min(threads, len(wl.queries)))
    qs = wl.queries[1:1 + nq].astype(np.float64) if len(wl.queries) > nq else wl.queries[:nq].astype(np.float64)
    t0 = time.perf_counter()
    _, used = O.nn_search_batch(qs, cands64, params, advanced, wl.dim_range, n_threads=threads)
    wall = time.perf_counter() - t0
    return {"value": len(qs) / wall, "unit": "queries/s", "cores": int(used), "kind": "port",
            "host_cpu": host_cpu(),
            "sample": f"{len(qs)} queries x {len(wl.candidates)} candidates, method {method}"
                      f"{'/' + advanced if advanced else ''}, W={w}, C port of mvdtw.nn_search "
                      f"(oracle/tcdtw_oracle.c), OpenMP over queries",
            "wall_s": wall}


def cpu_tc_dtw(wl, w, budget_s):
    """the CPU path also timed for tc_dtw, resolved as
    the reference CLI does (cli.py:228-235: tune_params + tc_dtw_select on the
    seeded sample, work model; untimed), then searched on a bounded sample."""
    from oracle import oracle as O

    e_ti, e_pc, lv, adv = O.resolve_tc_dtw(wl.queries.astype(np.float64), wl.candidates.astype(np.float64), w,
                                           wl.dim_range, seed=42)
    out = cpu_queries_per_sec(wl, w, "tc_dtw", adv, 0, budget_s,
                              knobs={"trigger_ti": e_ti, "trigger_pc": e_pc, "quant_levels": lv})
    out["resolved"] = {"advanced": adv, "trigger_ti": e_ti, "trigger_pc": e_pc, "quant_levels": lv}
    return out


# ----------------------------------------------------------------- main arms
def resolve_method(P, wl, w, method, dim_range):
    """The reference CLI's setup stage (cli.py:228-235): tune_params and,
    for tc_dtw, tc_dtw_select on the seeded sample; untimed."""
    if method == "auto":  # GPU-cost choice among LB_MV / TC-DTW(LB_PC) / TC-DTW(LB_TI) (row f1)
        base = P.tune_params(list(wl.queries[:64].astype(np.float64)), list(wl.candidates[:4096].astype(np.float64)),
                             P.SearchParams(window=w, method=P.Method.TC_DTW), seed=0, dim_range=dim_range,
                             metric="time")
        return P.select_method(list(wl.queries[:64].astype(np.float64)),
                               list(wl.candidates[:4096].astype(np.float64)), base, dim_range=dim_range)
    params = P.SearchParams(window=w, method=P.Method(method))
    advanced = None
    if params.method == P.Method.TC_DTW:
        params = P.tune_params(list(wl.queries[:64].astype(np.float64)), list(wl.candidates[:4096].astype(np.float64)),
                               params, seed=0, dim_range=dim_range)
        rng = np.random.default_rng(0)
        sq = [wl.queries[i].astype(np.float64) for i in sorted(rng.choice(len(wl.queries), 8, replace=False))]
        sc = [wl.candidates[i].astype(np.float64) for i in sorted(rng.choice(len(wl.candidates), 23, replace=False))]
        advanced = P.tc_dtw_select(sq, sc, params, dim_range=dim_range)
    elif params.method in (P.Method.LB_TI, P.Method.LB_PC, P.Method.LB_AD):
        params = P.tune_params(list(wl.queries[:64].astype(np.float64)), list(wl.candidates[:4096].astype(np.float64)),
                               params, seed=0, dim_range=dim_range)
    return params, advanced


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from paper_2101_07731_b200.datasets import make_workload
    import paper_2101_07731_b200.core as core

    wl = make_workload(args.config, n_candidates=args.candidates or None, n_queries=args.queries or None)
    w = wl.spec.windows()[args.window_index]
    method, advanced, knobs = args.method, None, {}
    if method == "auto":  # the reference has no GPU-cost choice: its classic bound
        method = "lb_mv"
    del core
    from oracle import oracle as O

    cands64 = wl.candidates.astype(np.float64)
    if method == "tc_dtw":  # resolved as the reference CLI does (cli.py:228-235), untimed
        e_ti, e_pc, lv, advanced = O.resolve_tc_dtw(wl.queries.astype(np.float64), cands64, w, wl.dim_range, seed=42)
        knobs = {"trigger_ti": e_ti, "trigger_pc": e_pc, "quant_levels": lv}
    params = O.make_params(w, method, **knobs)
    threads = os.cpu_count() or 1
    t0 = time.perf_counter()
    O.nn_search_batch(wl.queries[:1].astype(np.float64), cands64, params, advanced, wl.dim_range, n_threads=1)
    per_query = time.perf_counter() - t0
    # each step: one query per thread (bounded sample), so the run stays short
    nq = max(1, min(len(wl.queries), threads))
    times = []
    for s in range(args.warmup + args.steps):
        sel = (np.arange(nq) + s * nq) % len(wl.queries)
        qs = wl.queries[sel].astype(np.float64)
        t0 = time.perf_counter()
        O.nn_search_batch(qs, cands64, params, advanced, wl.dim_range, n_threads=threads)
        if s >= args.warmup:
            times.append(time.perf_counter() - t0)
    step = statistics.median(times)
    value = nq / step
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "queries/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": step * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, SURVEY 8d)",
        "config": {"workload": args.config, "n_candidates": len(wl.candidates), "n_queries_per_step": nq,
                   "window": w, "method": method, "advanced": advanced},
        "cpu_baseline": {"value": value, "unit": "queries/s", "cores": threads, "kind": "port", "host_cpu": host_cpu(),
                         "sample": f"{nq} queries/step x {len(wl.candidates)} candidates (C port of "
                                   f"mvdtw.nn_search, oracle/; single-query probe {per_query:.2f}s)"},
        "e2e": {"value": value, "unit": "queries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_ours(args):
    import torch

    rank, world, local = dist_env()
    if world > 1:
        import torch.distributed as dist

        if args.dist_backend == "nccl":  # the init log lets the driver verify the rank count
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")

        dev = local if args.dist_backend == "nccl" else local % torch.cuda.device_count()
        torch.cuda.set_device(dev)
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            dist.init_process_group(args.dist_backend)
    else:
        torch.cuda.set_device(0)
    import paper_2101_07731_b200 as P
    from paper_2101_07731_b200 import _lib
    from paper_2101_07731_b200.datasets import make_workload
    from paper_2101_07731_b200.distributed import combine_results, exchange_dbest, shard_bounds

    t_gen = time.perf_counter()
    wl = make_workload(args.config, n_candidates=args.candidates or None, n_queries=args.queries or None)
    t_gen = time.perf_counter() - t_gen
    w = wl.spec.windows()[args.window_index]
    n_total = len(wl.candidates)
    a, b = shard_bounds(n_total, world, rank)
    params, advanced = resolve_method(P, wl, w, args.method, wl.dim_range)
    t_up = time.perf_counter()
    index = P.SearchIndex(wl.candidates[a:b], dtype=wl.dtype, base=a)
    index.cascade = not args.no_cascade
    torch.cuda.synchronize()
    t_up = time.perf_counter() - t_up
    env_stats = index_envelope_stats(index, w, _lib)
    Qdev = index.prepare_queries(wl.queries)
    n_q = Qdev.shape[0]
    batch = args.batch or index.auto_batch(params, advanced, n_q, seeds=args.seeds, reverse_bound=args.reverse_bound)
    if world > 1:  # every rank must run the same batches (one d_best exchange per batch)
        bt = torch.tensor([batch], dtype=torch.int64, device="cuda")
        torch.distributed.all_reduce(bt, op=torch.distributed.ReduceOp.MIN)
        batch = int(bt.item())
    group = None
    hook = None
    if world > 1 and not args.no_exchange:
        hook = lambda d: exchange_dbest(d, group)  # noqa: E731

    def step(queries, to_host=False):
        res = index.search(queries, params, advanced=advanced, dim_range=wl.dim_range, batch=batch,
                           seeds=args.seeds, dbest_hook=hook, return_device=True,
                           reverse_bound=args.reverse_bound, reverse_pc=args.reverse_pc)
        idx, dist_ = res.best_index, res.best_distance
        if world > 1:
            idx, dist_ = combine_results(idx, dist_, group)
        if to_host:
            idx, dist_ = idx.cpu(), dist_.cpu()
        return idx, dist_, res

    def timed(fn, k):
        times = []
        for _ in range(k):
            if world > 1:
                torch.distributed.barrier()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1)
            if world > 1:
                t = torch.tensor([ms], device="cuda", dtype=torch.float64)
                torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
                ms = float(t.item())
            times.append(ms)
        return times

    L = _lib.load_library()
    for _ in range(args.warmup):
        step(Qdev)
    torch.cuda.synchronize()
    launches0 = L.tcdtw_launch_count() if hasattr(L, "tcdtw_launch_count") else 0
    with ClockSampler(torch.cuda.current_device()) as clk:
        times = timed(lambda: step(Qdev), args.steps)
    launches = (L.tcdtw_launch_count() - launches0) if hasattr(L, "tcdtw_launch_count") else None
    clocks = clk.summary()
    ms_step = statistics.median(times)
    value = n_q / (ms_step / 1e3)

    # end to end through the public API: pinned host queries in, host results out
    Qhost = torch.from_numpy(np.ascontiguousarray(wl.queries)).pin_memory()
    e2e_times = timed(lambda: step(Qhost, to_host=True), max(1, min(3, args.steps)))
    e2e_ms = statistics.median(e2e_times)

    # instrumented pass: phase times (CUDA events per phase), counters
    res = index.search(Qdev, params, advanced=advanced, dim_range=wl.dim_range, batch=batch, seeds=args.seeds,
                       timing=True, dbest_hook=hook, return_device=True, reverse_bound=args.reverse_bound,
                       reverse_pc=args.reverse_pc)
    ph = res.phase_ms
    ctr = {k: v.sum().item() for k, v in res.counters.items()}
    if world > 1:
        vec = torch.tensor([ctr[k] for k in _lib.COUNTERS], dtype=torch.float64, device="cuda")
        torch.distributed.all_reduce(vec)
        ctr = dict(zip(_lib.COUNTERS, vec.tolist()))
        pv = torch.tensor([ph[k] for k in _lib.PHASES], dtype=torch.float64, device="cuda")
        torch.distributed.all_reduce(pv, op=torch.distributed.ReduceOp.MAX)
        ph = dict(zip(_lib.PHASES, pv.tolist()))

    # ALU issue-rate probe (FP32 FFMA, independent chains) on this box
    lane_ops = __import__("ctypes").c_double()
    # the DTW arithmetic type's FMA rate (FP64 issues at half the FP32 rate)
    dtw_f32 = wl.dtype == "f32" or index.f32_filter  # float64 data under the float32 filter
    probe_dt = 0 if dtw_f32 else 1
    sink = torch.empty(1, device="cuda", dtype=torch.float64)
    L.tcdtw_alu_probe(probe_dt, 148 * 8, 2000, sink.data_ptr(), __import__("ctypes").byref(lane_ops),
                      _lib.stream_ptr())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    L.tcdtw_alu_probe(probe_dt, 148 * 8, 2000, sink.data_ptr(), __import__("ctypes").byref(lane_ops),
                      _lib.stream_ptr())
    e1.record()
    torch.cuda.synchronize()
    alu_peak = lane_ops.value / (e0.elapsed_time(e1) / 1e3) / 1e12  # T lane-op/s

    n, d = wl.spec.length, wl.spec.dims
    shard_n = b - a
    # L(5d+2) per pair as max(c-u, l-c, 0)^2; the float32 pass evaluates a term as
    # sat(|c-m| - h)^2 (FADD, FADD.SAT, FFMA): L(3d+2) issued -- the roofline counts what is issued
    lbmv_sat = dtw_f32 and not args.reverse_bound
    lbmv_ops = float(n_q) * shard_n * n * ((3 if lbmv_sat else 5) * d + 2)
    lbmv_bytes = (shard_n + 3 * n_q) * n * d * (4 if wl.dtype == "f32" else 8)
    dtw_cells = ctr["dtw_cells"]
    dtw_ms = ph["dtw"] + ph["seeds_dtw"]
    gcups = dtw_cells / (dtw_ms / 1e3) / 1e9 if dtw_ms > 0 else None
    dom = max(ph, key=ph.get)
    if dom == "lb_mv":
        achieved = lbmv_ops / (ph["lb_mv"] / 1e3) / 1e12
        roof = {"kernel": "lbmv_matrix_kernel", "bound": "alu", "achieved": achieved, "peak": alu_peak,
                "unit": "Tlane-op/s", "frac": achieved / alu_peak,
                "traffic": None, "algorithmic_ops_per_launch_set": lbmv_ops,
                "hbm_view": {"unique_bytes": lbmv_bytes,
                             "achieved_gbs": lbmv_bytes / (ph["lb_mv"] / 1e3) / 1e9,
                             "peak_gbs": measured_peaks().get("hbm_gbs")}}
    else:
        ops = dtw_cells * (2 * d + 4)
        achieved = ops / (dtw_ms / 1e3) / 1e12
        roof = {"kernel": index.dtw_kernel(params, advanced, batch), "bound": "alu", "achieved": achieved, "peak": alu_peak,
                "unit": "Tlane-op/s", "frac": achieved / alu_peak, "traffic": traffic_from_profile(dtw_cells / max(1, -(-n_q // batch))),
                "algorithmic_ops": f"(2d+4) = {2 * d + 4} per DP cell x {dtw_cells:.4g} cells (SURVEY 8d)"}
    if dom != "lb_mv" and ph.get("lb_mv", 0.0) > 0:
        mv_ach = lbmv_ops / (ph["lb_mv"] / 1e3) / 1e12
        roof["lb_mv"] = {"kernel": "lbmv_matrix_kernel" + ("<SAT>" if lbmv_sat else ""), "bound": "alu",
                         "achieved": mv_ach, "peak": alu_peak, "frac": mv_ach / alu_peak, "ms": ph["lb_mv"],
                         "ops_per_pair": n * ((3 if lbmv_sat else 5) * d + 2)}
    if ph.get("advanced", 0.0) > 0 and ctr.get("advanced_lb_evals", 0) > 0 and advanced is not None:
        # the second-stage bound's kernel against the same ALU roof, SURVEY 8(d) op counts per evaluated pair
        a_name = getattr(advanced, "value", str(advanced))
        if a_name == "lb_pc":
            per_pair = n * (5 * params.max_boxes * d + params.max_boxes + 2)
        else:  # lb_ti
            per_pair = n * ((2 * w + 1) * 10 + 2 * d + (2 * w + 1) * (2 * d + 1) / params.refresh_period)
        a_ach = ctr["advanced_lb_evals"] * per_pair / (ph["advanced"] / 1e3) / 1e12
        roof["advanced"] = {"kernel": "advanced_pc_kernel" if a_name == "lb_pc" else "advanced_kernel (LB_TI)",
                            "bound": "alu", "achieved": a_ach, "peak": alu_peak, "frac": a_ach / alu_peak,
                            "ops_per_pair": per_pair, "pairs": ctr["advanced_lb_evals"], "ms": ph["advanced"],
                            "note": "full-length op count; the cascade stops most pairs early, so frac "
                                    "understates the kernel's issue rate"}
    lanes = 128 if dtw_f32 else 64
    nominal = 148 * lanes * measured_peaks().get("sm_max_mhz", 1965) / 1e6
    roof["peak_source"] = (f"tcdtw_alu_probe {'FFMA' if dtw_f32 else 'DFMA'} issue rate measured in this "
                           f"run (nominal 148 SM x {lanes} lanes x {measured_peaks().get('sm_max_mhz', 1965)} MHz = "
                           f"{nominal:.1f} T)")
    roof["frac_of_nominal"] = roof["achieved"] / nominal
    roof["arithmetic"] = ("float32 filter on float64 inputs + float64 finalist re-score" if index.f32_filter
                          else ("float32 filter + float64 finalist re-score" if wl.dtype == "f32" else "float64"))

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        adv_name = None if advanced is None else advanced.value
        cpu = cpu_queries_per_sec(wl, w, params.method.value, adv_name, 0, args.cpu_seconds)
        if params.method.value != "tc_dtw":
            cpu["tc_dtw"] = cpu_tc_dtw(wl, w, args.cpu_seconds)

    if rank == 0:
        q_bytes = Qhost.numel() * Qhost.element_size()
        line = {
            "metric": METRIC, "value": value, "unit": "queries/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": wl.dtype, "data": "synthetic (seeded generator, SURVEY 8d; UCR absent)",
            "config": {"workload": args.config, "n_candidates": n_total, "n_queries": n_q, "length": n, "dims": d,
                       "window": w, "method": params.method.value,
                       "advanced": None if advanced is None else advanced.value,
                       "trigger_ti": params.trigger_ti, "trigger_pc": params.trigger_pc,
                       "quant_levels": params.quant_levels, "query_batch": batch,
                       "reverse_bound": bool(args.reverse_bound), "cascade": not args.no_cascade,
                       "reverse_pc": bool(args.reverse_pc),
                       "parallelism": f"candidate shards x{world}",
                       "l2": "inputs larger than L2 (collection resident in HBM, no flush)"},
            "e2e": {"value": n_q / (e2e_ms / 1e3), "unit": "queries/s", "h2d_bytes_per_step": q_bytes,
                    "d2h_bytes_per_step": n_q * 16},
            "gpu_launches": launches,
            "gcups": gcups, "dtw_cells": dtw_cells,
            "counters": {k: ctr[k] for k in _lib.COUNTERS},
            "phase_ms": ph,
            "roofline": roof,
            "index_envelope": env_stats,
            "clocks": clocks,
            "cpu_baseline": cpu,
            "setup_s": {"generate": t_gen, "upload": t_up},
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
