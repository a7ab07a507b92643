#!/usr/bin/env python
"""Benchmark of the SpTRSV hot path (arXiv 1710.04985) on B200.

python bench.py [--gpus N] [--steps K] [--warmup W] [--config 2] [--algo self]
                [--impl ours|reference]

A step is one solve of the configuration's triangular system(s) on an
analyzed handle (the setup phase is timed separately, as in the paper's
Tables 4-6, and reported as config.analysis_ms).  Inputs are seeded synthetic
matrices of the paper's workload shapes (workloads/).  Timing: W >= 3 warm-up
steps, then exactly K steps between barrier + synchronize; each solve is
bracketed by CUDA events on the launching stream and the L2 is flushed (a
256 MiB write, outside the events) before every timed solve.  Multi-GPU:
one process per GPU (torchrun), each rank solves its own independent RHS
(weak scaling; config 5 partitions 64 RHS, strong scaling), the time is the
max over ranks.

Metric (BASELINE.json): effective HBM GB/s per solve = compulsory bytes /
time, bytes = 4(n+1) + (4+s)nnz(T) + 2 s n nrhs; GFLOP/s
= nrhs (2 #offdiag + n_div) / time is reported beside it.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

FALLBACK_HBM_GBS = 6650.0          # B200_PROFILING.md fallback, used only without MEASURED_PEAKS.json
NOMINAL_HBM_GBS = 8000.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", type=int, default=2, choices=[1, 2, 3, 4, 5, 6],
                    help="1-5: BASELINE.json configs; 6: NEXT-4 independent block-Jacobi ILU(0) factors over the ranks")
    ap.add_argument("--algo", default="auto", choices=["self", "level", "block", "slfc", "levc", "small", "auto"],
                    help="auto: SMALL if the triangle fits one CTA's shared memory, else BLOCK on detected "
                         "5-/7-point grids, else SELF")
    ap.add_argument("--dtype", default="f64", choices=["f64", "f32"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-flush", action="store_true")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=10.0, help="seconds of oracle work for cpu_baseline")
    ap.add_argument("--extra", action="store_true", help="also time the other algos and print them")
    ap.add_argument("--no-cusparse", action="store_true", help="skip the cuSPARSE SpSV context timing")
    ap.add_argument("--streams", type=int, default=4, help="config 6: concurrent streams for the independent factors")
    return ap.parse_args()


# ------------------------------------------------------------------ process group
def init_ranks():
    """One process per GPU (torchrun): RANK / LOCAL_RANK / WORLD_SIZE from the
    environment.  NCCL when every rank has its own GPU (the driver's
    8-GPU runs); when ranks share a GPU (a test run of the multi-rank path on
    one device) the control-plane collectives -- a barrier before and scalar
    MAX / SUM reductions after the timed region, never on the solve path --
    use gloo on CPU tensors."""
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    ndev = max(1, torch.cuda.device_count())
    dev_index = local % ndev
    torch.cuda.set_device(dev_index)
    dev = torch.device("cuda", dev_index)
    backend = None
    if world > 1:
        backend = "nccl" if world <= ndev else "gloo"
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")
    return world, rank, local, dev, backend


def reduce_values(vals, op, backend, dev):
    """MAX or SUM over ranks of a few float64 scalars (outside the timed region)."""
    import torch
    import torch.distributed as dist
    t = torch.tensor(vals, dtype=torch.float64, device=dev if backend == "nccl" else "cpu")
    if backend is not None:
        dist.all_reduce(t, op=dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.SUM)
    return [float(v) for v in t.tolist()]


# ------------------------------------------------------------------ workload
def build_problem(cfg: int, rank: int, world: int):
    """Matrix + RHS of a configuration (identical on every rank: seeded).
    Returns dict with the CSR, solve list [(uplo, diag)], rhs and work counts."""
    import workloads
    m, p = workloads.config(cfg)
    if cfg == 3:
        solves = [("lower", "unit"), ("upper", "non_unit")]
    else:
        solves = [(p["uplo"], p["diag"])]
    if cfg == 5:
        from paper_1710_04985_b200 import partition
        a, b = partition.block_range(64, world, rank)
        rhs = workloads.rhs_columns(m.n, range(a, b))
        scaling = "strong"
    else:
        rhs = workloads.rhs(m.n, 1, seed=p["seed"] + 7919 * rank)
        scaling = "weak"
    return {"m": m, "solves": solves, "rhs": rhs, "scaling": scaling, "params": p}


def counts_from(n, offd, diag, nrhs, esize):
    """Compulsory bytes and flops of ONE solve (reading Q13):
    bytes = 4(n+1) + (4+s) nnz(T) + 2 s n nrhs, flops = nrhs (2 #offdiag + n_div),
    nnz(T) = #offdiag + n_div (n_div = n for NON_UNIT, 0 for UNIT)."""
    ndiv = n if diag == "non_unit" else 0
    return 4 * (n + 1) + (4 + esize) * (offd + ndiv) + 2 * esize * n * nrhs, nrhs * (2 * offd + ndiv)


def handle_counts(infos, solves, n, nrhs, esize):
    """Per-solve (bytes, flops) from the GPU analysis of each handle (its
    referenced off-diagonal count, info.nnz_used): the product path never
    calls the oracle."""
    return [counts_from(n, i["nnz_used"], diag, nrhs, esize) for i, (_, diag) in zip(infos, solves)]


def oracle_counts(m, solves, nrhs, esize):
    """The same counts for the reference (CPU oracle) arm, from oracle.select."""
    import oracle
    per = [counts_from(m.n, oracle.select(m, uplo, diag)["nnz_used"], diag, nrhs, esize) for uplo, diag in solves]
    return sum(p[0] for p in per), sum(p[1] for p in per)


ALGO_NAMES = {0: "self", 1: "level", 2: "block", 5: "slfc", 6: "levc", 7: "small"}


def kernel_of(info, nrhs):
    """(dominant kernel, launches per solve) of a handle's solve path (solve.cu,
    block.cu, column.cu, mrt.cu -- the selection rules of solve.cu's launch()):
    SELF and the <= 16-column multi-RHS kernel also launch k_prefill (x :=
    sentinel)."""
    algo = ALGO_NAMES.get(info["algo"], "self")
    if nrhs == 1:
        return {"self": ("k_self", 2), "level": ("k_level", 1), "block": ("k_block", 1),
                "slfc": ("k_slfc", 1), "levc": ("k_levc", 1), "small": ("k_small", 1)}[algo]
    if nrhs <= 16 and algo not in ("level", "levc"):
        return ("k_mrhs_vf", 2)
    es = 8 if info["dtype"] == 0 else 4
    if algo not in ("level", "levc") and info["max_row_deps"] <= 4 and (nrhs * es) % 16 == 0:
        return ("k_mrt", (nrhs + 63) // 64)          # multi-RHS tile kernel (mrt.cu; aligned torch buffers)
    return ("k_level_mrhs", (nrhs + 127) // 128)


def break_even_solves(setup_ours, solve_ours, setup_other, solve_other):
    """Table 7's n_s: the smallest number of solves n >= 1 with
    setup_ours + n solve_ours < setup_other + n solve_other; None if there is
    none (our solve is not faster and our setup is not cheaper)."""
    if setup_ours + solve_ours < setup_other + solve_other:
        return 1
    if solve_ours >= solve_other:
        return None
    n = int((setup_ours - setup_other) // (solve_other - solve_ours)) + 1
    while setup_ours + n * solve_ours >= setup_other + n * solve_other:     # floating-point edge
        n += 1
    return max(n, 1)


def build_digest():
    """sha256 of the library's sources and nvcc flags (build.source_digest)."""
    from paper_1710_04985_b200 import build as B
    try:
        return B.source_digest()
    except OSError:
        return None


def lib_sha256():
    import hashlib
    from paper_1710_04985_b200 import build as B
    try:
        with open(B.LIB, "rb") as f:
            return hashlib.sha256(f.read()).hexdigest()
    except OSError:
        return None


def host_cpu():
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"model": model, "logical_cores": os.cpu_count()}


def measured_peak():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def ncu_traffic(key, sha):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of the dominant
    kernel, from an ncu --set full capture of THIS library build (entries are
    keyed by config/kernel/dtype and carry the build digest -- sha256 of the
    sources and nvcc flags -- they were measured on; any other build -> None)."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            ent = json.load(f).get(key)
    except Exception:
        return None
    if not isinstance(ent, dict) or sha is None or ent.get("build_digest") != sha:
        return None
    return ent.get("bytes")


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """SM clocks + throttle reasons sampled DURING the timed region: NVML polled
    every ~1 ms from a thread (a cfg2 timed region lasts ~10 ms, shorter than
    nvidia-smi's 20 ms loop); nvidia-smi -lms 20 if NVML is unavailable."""

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.rows = []
        self.proc = None
        self.nvml = None
        self.stop = False
        self.thread = None

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.gpu)
            mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            bits = [pynvml.nvmlClocksEventReasonHwSlowdown, pynvml.nvmlClocksEventReasonHwThermalSlowdown,
                    pynvml.nvmlClocksEventReasonSwThermalSlowdown, pynvml.nvmlClocksEventReasonSwPowerCap]
            self.nvml = pynvml

            def poll():
                while not self.stop:
                    sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                    rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                    self.rows.append([str(sm), str(mx), "", ""] +
                                     ["Active" if rs & bit else "Not Active" for bit in bits])
                    time.sleep(0.001)
            self.thread = threading.Thread(target=poll, daemon=True)
            self.thread.start()
            t0 = time.time()
            while not self.rows and time.time() - t0 < 3.0:   # sampler running before the region
                time.sleep(0.001)
            self.rows.clear()
            return self
        except Exception:
            self.nvml = None
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "20"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
            t0 = time.time()
            while not self.rows and time.time() - t0 < 3.0:   # sampler running before the region
                time.sleep(0.01)
            self.rows.clear()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 8:
                self.rows.append(parts)

    def __exit__(self, *a):
        self.stop = True
        if self.nvml is not None and self.thread is not None:
            self.thread.join(timeout=1)
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[4 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows), "source": "nvml" if self.nvml else "nvidia-smi"}


# ------------------------------------------------------------------ CPU oracle legs
def time_oracle(m, solves, rhs, budget_s, min_reps=1, max_reps=None):
    """Repeat the oracle's full solves (the whole workload, single-threaded C)
    until ``budget_s`` seconds of CPU work; returns (seconds per step, reps)."""
    import oracle
    reps = 0
    t0 = time.perf_counter()
    while True:
        z = rhs
        for uplo, diag in solves:
            z = oracle.solve(m, z, uplo, diag)
        reps += 1
        el = time.perf_counter() - t0
        if (el >= budget_s and reps >= min_reps) or (max_reps and reps >= max_reps):
            break
    return el / reps, reps


def run_reference(args):
    """--impl reference: this tier's reference arm is the CPU oracle as it
    stands, timed on the host cores on the same config/metric."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.config == 6:
        return run_reference_blocks(args, world)
    prob = build_problem(args.config, 0, 1)
    m, solves, rhs = prob["m"], prob["solves"], prob["rhs"]
    esize = 8 if args.dtype == "f64" else 4
    nbytes, flops = oracle_counts(m, solves, rhs.shape[1], esize)
    # warmup W untimed steps, then K timed steps (each = the full solve, bounded by the workload)
    for _ in range(args.warmup):
        time_oracle(m, solves, rhs, 0.0, max_reps=1)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        time_oracle(m, solves, rhs, 0.0, max_reps=1)
    per = (time.perf_counter() - t0) / max(1, args.steps)
    value = nbytes / per / 1e9
    line = {
        "impl": "reference", "metric": "SpTRSV effective HBM GB/s per solve (fraction of B200 peak)",
        "value": round(value, 4), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(per * 1e3, 4), "higher_is_better": True,
        "scaling": prob["scaling"], "vs_baseline": None, "dtype": args.dtype, "data": "synthetic",
        "gflops": round(flops / per / 1e9, 4),
        "config": {"workload": config_name(args.config, args.dtype), "n": m.n, "nrhs": int(rhs.shape[1]),
                   "bytes_per_step": nbytes, "flops_per_step": flops},
        "cpu_baseline": {"value": round(value, 4), "unit": "GB/s", "cores": 1, "kind": "oracle",
                         "sample": f"{args.steps} full oracle solves of {config_name(args.config, args.dtype)}",
                         "host": host_cpu()},
        "e2e": {"value": round(value, 4), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_reference_blocks(args, world):
    """--impl reference for config 6: the oracle's pair solves of all 16
    factors (bounded: each step is the whole batch)."""
    import workloads
    blocks, p = workloads.config(6)
    esize = 8 if args.dtype == "f64" else 4
    nbytes = flops = 0
    for b in blocks:
        for uplo, diag in (("lower", "unit"), ("upper", "non_unit")):
            by, fl = oracle_counts(b, [(uplo, diag)], 1, esize)
            nbytes += by
            flops += fl
    rhs = [workloads.rhs(b.n, 1, seed=p["seed"] + i)[:, 0] for i, b in enumerate(blocks)]

    def step():
        for b, r in zip(blocks, rhs):
            time_oracle(b, [("lower", "unit"), ("upper", "non_unit")], r, 0.0, max_reps=1)

    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    per = (time.perf_counter() - t0) / max(1, args.steps)
    value = nbytes / per / 1e9
    print(json.dumps({
        "impl": "reference", "metric": "SpTRSV effective HBM GB/s per solve (fraction of B200 peak)",
        "value": round(value, 4), "unit": "GB/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(per * 1e3, 4), "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": args.dtype, "data": "synthetic", "gflops": round(flops / per / 1e9, 4),
        "config": {"workload": "cfg6 (NEXT-4): 16 block-Jacobi ILU(0) factors, Eq. (3) pair each",
                   "bytes_per_step": nbytes, "flops_per_step": flops},
        "cpu_baseline": {"value": round(value, 4), "unit": "GB/s", "cores": 1, "kind": "oracle",
                         "sample": f"{args.steps} oracle pair solves of all 16 factors", "host": host_cpu()},
        "e2e": {"value": round(value, 4), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}),
        flush=True)


def config_name(cfg, dtype="f64"):
    p = {"f64": "fp64", "f32": "fp32"}[dtype]
    return {1: f"cfg1: L+D of 2D 5-point 32x32, {p}, 1 RHS",
            2: f"cfg2: L+D of 3D 7-point 128^3 (n=2097152), {p}, 1 RHS",
            3: f"cfg3: ILU(0) of 3D 27-point 96^3, forward (unit L) + backward (U) solve, {p}",
            4: f"cfg4: generated power-law lower factor n=4194304 nlev=12288, {p}",
            5: f"cfg5: 64 RHS on the 3D 7-point 128^3 factor, column-partitioned over ranks, {p}"}[cfg]


def latency_per_level(S, algo, dt, dev):
    """Measured time per dependent level of `algo` when nothing but the chain
    runs: BLOCK on one 8x4-column warp tile of a 7-point grid (one step per
    level), the row-wise algorithms on a bidiagonal chain (one row per level).
    nlev x this is the latency floor of a solve."""
    import torch
    import workloads
    if algo == "block":
        m = workloads.stencil((8, 4, 1024), 7, "lower")
    else:
        n = 4096
        rp = np.arange(0, 2 * n, 2, dtype=np.int32) - 1
        rp[0] = 0
        rp = np.append(rp, 2 * n - 1).astype(np.int32)
        ci = np.empty(2 * n - 1, dtype=np.int32)
        ci[0] = 0
        ci[1::2] = np.arange(0, n - 1)
        ci[2::2] = np.arange(1, n)
        va = np.empty(2 * n - 1)
        va[0] = 1.0
        va[1::2] = -0.5
        va[2::2] = 1.0
        m = workloads.CSR(n, rp, ci, va)
    h = S.from_csr(m, dtype=dt, algo=algo)
    nlev = h.info()["nlev"]
    bb = torch.ones(m.n, dtype=dt, device=dev)
    xx = torch.empty_like(bb)
    for _ in range(3):
        h.solve(bb, xx)
    torch.cuda.synchronize()
    ts = []
    for _ in range(10):
        a_, e_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a_.record()
        h.solve(bb, xx)
        e_.record()
        e_.synchronize()
        ts.append(a_.elapsed_time(e_) * 1e-3)
    return float(np.median(ts)) / nlev, {"probe": f"{'8x4x1024 7-point tile' if algo == 'block' else 'chain n=4096'}",
                                         "nlev": nlev, "us": round(float(np.median(ts)) * 1e6, 2)}


def oracle_parity(m, solves, rhs_np, ours, dtype):
    """The timed step's output against the CPU oracle on the same input (all
    columns up to 4; else columns 0, middle, last): max relative error."""
    import oracle
    nrhs = rhs_np.shape[1]
    cols = list(range(nrhs)) if nrhs <= 4 else sorted({0, nrhs // 2, nrhs - 1})
    z = np.ascontiguousarray(rhs_np[:, cols])
    npdt = np.float64 if dtype == "f64" else np.float32
    mm = m.astype(npdt) if npdt is np.float32 else m
    for uplo, diag in solves:
        z = oracle.solve(mm, z.astype(npdt), uplo, diag, dtype=npdt)
    o = ours.reshape(m.n, -1)[:, cols].astype(np.float64)
    ref = np.asarray(z, dtype=np.float64).reshape(m.n, -1)
    err = float(np.abs(o - ref).max() / max(np.abs(ref).max(), 1e-300))
    tol = 1e-10 if dtype == "f64" else 1e-4
    return {"max_rel_err_vs_oracle": err, "tol": tol, "ok": bool(err <= tol), "columns": cols}


# ------------------------------------------------------------------ our arm
def run_ours(args):
    import torch
    import torch.distributed as dist
    from paper_1710_04985_b200 import sptrsv as S

    world, rank, local, dev, backend = init_ranks()

    prob = build_problem(args.config, rank, world)
    m, solves, rhs_np = prob["m"], prob["solves"], prob["rhs"]
    dt = torch.float64 if args.dtype == "f64" else torch.float32
    esize = 8 if args.dtype == "f64" else 4
    nrhs = rhs_np.shape[1]

    stream = torch.cuda.current_stream()
    # warm-up handle: CUDA module loading is not part of the analysis time
    import workloads
    _w = workloads.stencil((8, 8), 5, "lower")
    S.from_csr(_w, dtype=dt, algo=args.algo)
    # the CSR is uploaded first: the setup phase (analysis + the algorithm's
    # build) is timed on device-resident inputs, like cuSPARSE's analysis below
    d_rp = torch.from_numpy(np.ascontiguousarray(m.rowptr, dtype=np.int32)).to(dev)
    d_ci = torch.from_numpy(np.ascontiguousarray(m.colidx, dtype=np.int32)).to(dev)
    d_va = torch.from_numpy(np.ascontiguousarray(m.vals)).to(device=dev, dtype=dt)
    torch.cuda.synchronize()
    # the first setup of the process also grows the device memory pool: the
    # second one is timed (warm process, like cuSPARSE's below)
    handles = [S.TriangularSolver(m.n, d_rp, d_ci, d_va, uplo, diag, args.algo) for uplo, diag in solves]
    torch.cuda.synchronize()
    del handles
    t_an = time.perf_counter()
    handles = [S.TriangularSolver(m.n, d_rp, d_ci, d_va, uplo, diag, args.algo) for uplo, diag in solves]
    torch.cuda.synchronize()
    analysis_ms = (time.perf_counter() - t_an) * 1e3
    # numerical refactorization (NEXT-2): new values, same pattern
    t_up = time.perf_counter()
    for h in handles:
        h.update_values(d_rp, d_ci, d_va)
    torch.cuda.synchronize()
    update_ms = (time.perf_counter() - t_up) * 1e3
    del d_rp, d_ci, d_va
    an_infos = [h.info() for h in handles]
    per_solve = handle_counts(an_infos, solves, m.n, nrhs, esize)
    nbytes, flops = sum(p[0] for p in per_solve), sum(p[1] for p in per_solve)

    b = torch.from_numpy(np.ascontiguousarray(rhs_np[:, 0] if nrhs == 1 else rhs_np)).to(dev, dt)
    bufs = [torch.empty_like(b) for _ in handles]
    flush = None if args.no_flush else torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    def step():
        z = b
        for h, out in zip(handles, bufs):
            h.solve(z, out)
            z = out
        return z

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()

    # events bracket every step and every solve (one kernel each for BLOCK /
    # LEVEL; the per-solve times give the dominant kernel's launch duration)
    nh = len(handles)
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(nh + 1)] for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for k in range(args.steps):
            if flush is not None:
                flush.zero_()
            ev[k][0].record(stream)
            z = b
            for i, (h, out) in enumerate(zip(handles, bufs)):
                h.solve(z, out)
                z = out
                ev[k][i + 1].record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    times = np.array([e[0].elapsed_time(e[nh]) for e in ev]) / 1e3          # seconds per step
    solve_times = np.array([[e[i].elapsed_time(e[i + 1]) for i in range(nh)] for e in ev]) / 1e3
    t_mean = float(times.mean())
    t_med = float(np.median(times))
    t_max = reduce_values([t_mean], "max", backend, dev)[0]
    total_bytes = nbytes * (world if prob["scaling"] == "weak" else 1)
    total_flops = flops * (world if prob["scaling"] == "weak" else 1)
    if prob["scaling"] == "strong":
        # config 5: bytes counted per GPU (each replica streams the matrix), summed
        total_bytes, total_flops = reduce_values([nbytes, flops], "sum", backend, dev)
    value = total_bytes / t_max / 1e9

    # e2e through the C ABI with HOST buffers (pinned), H2D + D2H inside the region
    e2e = None
    if not args.no_e2e:
        hb = torch.from_numpy(np.ascontiguousarray(rhs_np[:, 0] if nrhs == 1 else rhs_np)).to(dt).pin_memory()
        hx = [torch.empty_like(hb).pin_memory() for _ in handles]
        for _ in range(3):
            z = hb
            for h, out in zip(handles, hx):
                h.solve_host(z, out)
                z = out
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        k_e2e = max(5, min(args.steps, 20))
        t0 = time.perf_counter()
        for _ in range(k_e2e):
            z = hb
            for h, out in zip(handles, hx):
                h.solve_host(z, out)
                z = out
        t_e2e = reduce_values([(time.perf_counter() - t0) / k_e2e], "max", backend, dev)[0]
        e2e = {"value": round(total_bytes / t_e2e / 1e9, 3), "unit": "GB/s",
               "h2d_bytes_per_step": int(hb.numel() * esize * len(handles)),
               "d2h_bytes_per_step": int(hb.numel() * esize * len(handles)),
               "ms_per_step": round(t_e2e * 1e3, 4), "api": "sptrsv_solve_host"}

    # cuSPARSE SpSV on the same problem, same protocol (context)
    cusp = None
    if not args.no_cusparse and world == 1:
        try:
            import baseline
            npdt = np.float64 if args.dtype == "f64" else np.float32
            cbufs = [torch.empty_like(b) for _ in handles]
            # warm-up context: cuSPARSE's module loading is not part of its analysis time
            _wb = torch.ones(64, dtype=dt, device=dev)
            _wx = torch.empty_like(_wb)
            baseline.CusparseSpSV(_w, "lower", "non_unit", _wb, _wx, npdt).solve(stream.cuda_stream)
            torch.cuda.synchronize()
            ctxs, z = [], b
            torch.cuda.synchronize()
            t_ca = time.perf_counter()
            Cls = baseline.CusparseSpSV if nrhs == 1 else baseline.CusparseSpSM     # SpSM for cfg5
            for (uplo, diag), out in zip(solves, cbufs):
                ctxs.append(Cls(m, uplo, diag, z, out, npdt))
                z = out
            torch.cuda.synchronize()
            cusp_an_ms = sum(c.analysis_ms for c in ctxs)        # cusparseSpSV_analysis, CUDA events
            sp = stream.cuda_stream
            for _ in range(3):
                for c in ctxs:
                    c.solve(sp)
            torch.cuda.synchronize()
            ts = []
            for _ in range(max(5, args.steps // 2)):
                if flush is not None:
                    flush.zero_()
                a_, e_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a_.record(stream)
                for c in ctxs:
                    c.solve(sp)
                e_.record(stream)
                e_.synchronize()
                ts.append(a_.elapsed_time(e_) / 1e3)
            tc = float(np.mean(ts))
            ours = bufs[-1].double()
            diff = float((cbufs[-1].double() - ours).abs().max() / ours.abs().max().clamp_min(1e-300))
            cusp = {"us_per_step": round(tc * 1e6, 2), "GB/s": round(nbytes / tc / 1e9, 2),
                    "speedup_ours": round(tc / t_mean, 3), "max_rel_diff_vs_ours": diff,
                    "analysis_ms": round(cusp_an_ms, 2),
                    "break_even_solves_vs_ours": break_even_solves(analysis_ms * 1e-3, t_mean, cusp_an_ms * 1e-3, tc),
                    "analysis_note": "cusparseSpSV_analysis / cusparseSpSM_analysis only (CUDA events); ours: wall clock of sptrsv_analyze + set_algo builds on device-resident CSR, warm process; break_even_solves_vs_ours = Table 7's n_s (P:1412-1420), null if none",
                    "api": ("cusparseSpSV_solve (CUSPARSE_SPSV_ALG_DEFAULT)" if nrhs == 1 else
                            f"cusparseSpSM_solve (CUSPARSE_SPSM_ALG_DEFAULT, {nrhs} row-major RHS)")
                           + ", analysis outside the timing"}
            del ctxs
        except Exception as e:              # context only: never fails the bench
            cusp = {"unavailable": str(e)[:200]}

    # extra: the other algorithms on the same problem (context, rank 0 prints)
    extra = {}
    if args.extra and world == 1:
        for algo in ("self", "level", "block", "slfc", "levc", "small"):
            if algo == args.algo:
                continue
            try:
                for h in handles:
                    h.set_algo(algo)
            except Exception as e:          # not available
                extra[algo] = str(e)
                continue
            for _ in range(3):
                step()
            torch.cuda.synchronize()
            ts = []
            for _ in range(max(5, args.steps // 2)):
                if flush is not None:
                    flush.zero_()
                a_, e_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a_.record(stream)
                step()
                e_.record(stream)
                e_.synchronize()
                ts.append(a_.elapsed_time(e_) / 1e3)
            tm = float(np.mean(ts))
            extra[algo] = {"us_per_step": round(tm * 1e6, 2), "GB/s": round(nbytes / tm / 1e9, 2)}
        for h in handles:
            h.set_algo(args.algo)

    out_np = bufs[-1].cpu().numpy() if rank == 0 else None
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    peak, peak_src = measured_peak()
    # dominant kernel: the solve with the largest mean time; achieved = its
    # algorithmic bytes / its mean launch duration (CUDA events on its stream)
    kinfo = [kernel_of(i, nrhs) for i in an_infos]
    dom = int(np.argmax(solve_times.mean(axis=0)))
    t_dom = float(solve_times[:, dom].mean())
    achieved = per_solve[dom][0] / t_dom / 1e9
    launches_per_step = sum(k[1] for k in kinfo)
    # cpu_baseline leg (the one place this arm executes oracle/): the oracle
    # timed on the host cores, and the timed step's output checked against it
    cpu = None
    if not args.no_cpu and world == 1:
        per, reps = time_oracle(m, solves, rhs_np, args.cpu_budget, min_reps=2)
        cpu = {"value": round(nbytes / per / 1e9, 4), "unit": "GB/s", "cores": 1, "kind": "oracle",
               "sample": f"{reps} full oracle solves of the same workload ({per * 1e3:.1f} ms each, "
                         f"~{args.cpu_budget:.0f} s budget), single-threaded C -O2",
               "host": host_cpu()}
    parity = oracle_parity(m, solves, rhs_np, out_np, args.dtype)
    dom_algo = ALGO_NAMES.get(an_infos[dom]["algo"], "self")
    try:
        t_lev, lev_probe = latency_per_level(S, dom_algo if nrhs == 1 else "self", dt, dev)
    except Exception as e:                 # never fails the bench
        t_lev, lev_probe = None, {"unavailable": str(e)[:120]}
    eff_algo = "+".join(sorted({ALGO_NAMES.get(i["algo"], "?") for i in an_infos}))
    key = f"cfg{args.config}_{kinfo[dom][0]}_{args.dtype}"
    sha = build_digest()
    clk_s = clk.summary()
    line = {
        "metric": "SpTRSV effective HBM GB/s per solve (fraction of B200 peak)",
        "value": round(value, 3), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
        "warmup": max(3, args.warmup), "ms_per_step": round(t_max * 1e3, 5),
        "higher_is_better": True, "scaling": prob["scaling"], "vs_baseline": None,
        "dtype": args.dtype, "data": "synthetic (seeded generators, workloads/)",
        "gflops": round(total_flops / t_max / 1e9, 3),
        "config": {"workload": config_name(args.config, args.dtype), "algo": args.algo, "algo_used": eff_algo,
                   "n": m.n, "nrhs": int(nrhs),
                   "nnz_used": [i["nnz_used"] for i in an_infos], "nlev": [i["nlev"] for i in an_infos],
                   "bytes_per_step": nbytes, "flops_per_step": flops,
                   "analysis_ms": round(analysis_ms, 2), "update_values_ms": round(update_ms, 2),
                   "l2": "flushed before every timed solve (256 MiB write)" if flush is not None else "warm",
                   "median_us": round(t_med * 1e6, 2), "min_us": round(float(times.min()) * 1e6, 2),
                   "parallelism": f"replicas{world}" if prob["scaling"] == "weak" else f"rhs-partition{world}"},
        "roofline": {"bound": "hbm", "achieved": round(achieved, 2), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "traffic": ncu_traffic(key, sha), "peak_source": peak_src,
                     "traffic_source": "profiles/ncu_traffic.json entry of this build (sha256 of its sources and nvcc flags), else null",
                     "frac_of_nominal": round(achieved / NOMINAL_HBM_GBS, 4),
                     "kernel": kinfo[dom][0], "kernel_us": round(t_dom * 1e6, 2),
                     "bytes_per_launch": int(per_solve[dom][0]),
                     "share_of_step": round(t_dom / t_mean, 4),
                     "nlev": an_infos[dom]["nlev"],
                     "ns_per_level_alone": round(t_lev * 1e9, 1) if t_lev else None,
                     "latency_floor_us": round(an_infos[dom]["nlev"] * t_lev * 1e6, 2) if t_lev else None,
                     "latency_floor_probe": lev_probe,
                     "ns_per_level_achieved": round(t_dom * 1e9 / max(1, an_infos[dom]["nlev"]), 1)},
        "parity": parity,
        "build_digest": sha, "lib_sha256": lib_sha256(),
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": int(args.steps * launches_per_step),
        "clocks": clk_s,
    }
    if extra:
        line["extra_algos"] = extra
    if cusp is not None:
        line["cusparse_spsv"] = cusp
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


# ------------------------------------------------------------ config 6 (NEXT-4)
def run_blocks(args):
    """Independent factors over the ranks (NEXT-4): 16 block-Jacobi ILU(0)
    factors (27-point 128^3 split into uneven z-slabs, workloads.block_jacobi_ilu0),
    assigned to ranks by partition.factor_assignment (LPT on nnz); a step is the
    Eq. (3) pair solve (unit L, then U) of every factor a rank owns, one RHS per
    factor.  No collective on the solve path; time = max over ranks; value = the
    compulsory bytes of all factors' pair solves / that time (strong scaling:
    the total work is fixed)."""
    import torch
    import torch.distributed as dist
    import workloads
    from paper_1710_04985_b200 import partition
    from paper_1710_04985_b200 import sptrsv as S
    world, rank, local, dev, backend = init_ranks()
    blocks, p = workloads.config(6)
    owned = partition.factor_assignment([int(b.rowptr[-1]) for b in blocks], world)[rank]
    dt = torch.float64 if args.dtype == "f64" else torch.float32
    esize = 8 if args.dtype == "f64" else 4
    t_an = time.perf_counter()
    items = []
    for i in owned:
        b = blocks[i]
        hl = S.from_csr(b, "lower", "unit", dtype=dt, algo=args.algo)
        hu = S.from_csr(b, "upper", "non_unit", dtype=dt, algo=args.algo)
        rhs = torch.from_numpy(workloads.rhs(b.n, 1, seed=p["seed"] + i)[:, 0]).to(dev, dt)
        items.append((i, hl, hu, rhs, torch.empty_like(rhs), torch.empty_like(rhs)))
    torch.cuda.synchronize()
    analysis_ms = (time.perf_counter() - t_an) * 1e3
    local_bytes = local_flops = 0
    for _, hl, hu, rhs, _, _ in items:
        for h, diag in ((hl, "unit"), (hu, "non_unit")):
            by, fl = counts_from(rhs.numel(), h.info()["nnz_used"], diag, 1, esize)
            local_bytes += by
            local_flops += fl
    flush = None if args.no_flush else torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    # the rank's factors are independent: their pair solves run concurrently on
    # a pool of streams (sptrsv.StreamBatch), --streams 1 = one after another
    batch = S.StreamBatch(args.streams)
    chains = [[(hl, rhs, y), (hu, y, x)] for _, hl, hu, rhs, y, x in items]

    def step():
        batch.run(chains)

    for _ in range(max(3, args.warmup)):
        step()
    stream = torch.cuda.current_stream()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for k in range(args.steps):
            if flush is not None:
                flush.zero_()
            ev[k][0].record(stream)
            step()
            ev[k][1].record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    t_mean = float(np.mean([a.elapsed_time(b) for a, b in ev])) / 1e3
    t_max = reduce_values([t_mean], "max", backend, dev)[0]
    total_bytes, total_flops = reduce_values([float(local_bytes), float(local_flops)], "sum", backend, dev)
    # e2e through the C ABI with host buffers
    hb = [it[3].cpu().pin_memory() for it in items]
    hy = [torch.empty_like(v).pin_memory() for v in hb]
    hx = [torch.empty_like(v).pin_memory() for v in hb]
    for (i, hl, hu, _, _, _), b_, y_, x_ in zip(items, hb, hy, hx):
        hl.solve_host(b_, y_)
        hu.solve_host(y_, x_)
    if world > 1:
        dist.barrier()
    k_e2e = max(3, min(args.steps, 10))
    t0 = time.perf_counter()
    for _ in range(k_e2e):
        for (i, hl, hu, _, _, _), b_, y_, x_ in zip(items, hb, hy, hx):
            hl.solve_host(b_, y_)
            hu.solve_host(y_, x_)
    t_e2e = reduce_values([(time.perf_counter() - t0) / k_e2e], "max", backend, dev)[0]
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    peak, peak_src = measured_peak()
    # cpu_baseline leg (the one place this arm executes oracle/): the oracle on
    # the owned factors, and the timed output of the first factor against it
    import oracle
    cpu = None
    i0, hl0, hu0, rhs0, _, x0 = items[0]
    b0 = blocks[i0]
    z = oracle.solve(b0, rhs0.double().cpu().numpy(), "lower", "unit")
    z = oracle.solve(b0, z, "upper", "non_unit")
    ref = np.asarray(z, dtype=np.float64)
    err = float(np.abs(x0.double().cpu().numpy() - ref).max() / np.abs(ref).max())
    parity = {"max_rel_err_vs_oracle": err, "tol": 1e-10 if args.dtype == "f64" else 1e-4,
              "ok": bool(err <= (1e-10 if args.dtype == "f64" else 1e-4)), "factor": i0}
    if not args.no_cpu and world == 1:
        reps, tc0 = 0, time.perf_counter()
        while time.perf_counter() - tc0 < args.cpu_budget:
            for i, _, _, rhs, _, _ in items:
                zz = oracle.solve(blocks[i], rhs.double().cpu().numpy(), "lower", "unit")
                oracle.solve(blocks[i], zz, "upper", "non_unit")
            reps += 1
        per = (time.perf_counter() - tc0) / reps
        cpu = {"value": round(local_bytes / per / 1e9, 4), "unit": "GB/s", "cores": 1, "kind": "oracle",
               "sample": f"{reps} oracle pair solves of all {len(items)} factors ({per * 1e3:.1f} ms each)",
               "host": host_cpu()}
    achieved = local_bytes / t_mean / 1e9
    line = {
        "metric": "SpTRSV effective HBM GB/s per solve (fraction of B200 peak)",
        "value": round(total_bytes / t_max / 1e9, 3), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
        "warmup": max(3, args.warmup), "ms_per_step": round(t_max * 1e3, 5), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": args.dtype,
        "data": "synthetic (seeded generators, workloads/)", "gflops": round(total_flops / t_max / 1e9, 3),
        "config": {"workload": "cfg6 (NEXT-4): 16 block-Jacobi ILU(0) factors of the 27-point 128^3 Laplacian "
                               f"(uneven z-slabs), Eq. (3) pair per factor, {args.dtype}",
                   "algo": args.algo, "factors_total": len(blocks), "factors_rank0": [it[0] for it in items],
                   "streams": args.streams,
                   "analysis_ms_rank0": round(analysis_ms, 2),
                   "l2": "flushed before every timed step (256 MiB write)" if flush is not None else "warm",
                   "parallelism": f"factor-partition{world} (LPT on nnz, no collective on the solve path)"},
        "roofline": {"bound": "hbm", "achieved": round(achieved, 2), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "traffic": None, "peak_source": peak_src,
                     "kernel": "all pair solves of rank 0 (SELF/AUTO kernels)", "bytes_per_step_rank0": local_bytes},
        "parity": parity, "cpu_baseline": cpu,
        "e2e": {"value": round(total_bytes / t_e2e / 1e9, 3), "unit": "GB/s",
                "h2d_bytes_per_step": int(sum(v.numel() for v in hb) * esize),
                "d2h_bytes_per_step": int(sum(v.numel() for v in hb) * esize),
                "ms_per_step": round(t_e2e * 1e3, 4), "api": "sptrsv_solve_host (pair per factor)"},
        "gpu_launches": int(args.steps * 2 * len(items) * (2 if args.algo in ("self", "auto") else 1)),
        "clocks": clk.summary(),
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    elif args.config == 6:
        run_blocks(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
