#!/usr/bin/env python
"""Benchmark of the CS-RBF normal-equation hot path (BASELINE.json metric:
A^T A assembly points/s and end-to-end fit time; fraction of the fp64 roofline).

  python bench.py [--gpus N --steps K --warmup W] [--config cfg5] [--impl reference]

Default workload: BASELINE config 5 (N = 2e8 Halton points, M = 1e6 grid
centres, wendland-3-1), the largest configuration that fits one B200.

* value  -- one step = bin + assemble A^T A / A^T h over the whole point set
  with the inputs resident in HBM (+ the NCCL all-reduce of the partial
  systems when N > 1); points/s over all ranks, max-over-ranks device time.
* e2e    -- the public fit through the C ABI (api.fit: rbg_create,
  rbg_set_centres, rbg_assemble from pageable host arrays, rbg_solve, c back
  to the host), a fresh context every step, so the centre grid, the symbolic
  pattern, the assembly layout and every host<->device copy are inside the
  timed region; points/s of the full fit.
* N > 1 is strong scaling: the one point set is split into equal-count spatial
  slabs (configs.slab_points), each rank bins and assembles only its slab
  against the replicated centres, and one in-place NCCL all-reduce sums
  [values | rhs | hits]; for e2e every rank then solves the summed system.

--impl reference times the reference's own CPU path (oracle/_ref: its
kd-tree, assemble_submatrix, transpose_matvec, gram_self compiled from
/root/reference; the dense Cholesky with the reference's ridge ladder on
OpenBLAS through scipy standing in for Eigen's LLT) on a spatial window of the
same workload -- every window point sees its full support -- using all host
threads (one reference instance per thread on point shards, partial systems
summed).  It loads no library of this package.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

METRIC = "A^T A assembly points/s"
UNIT = "points/s"
DEFAULT_CONFIG = "cfg5"
F_PHI = {2: 14, 3: 20}  # flops per phi evaluation incl. distance
FAMILY = {"wendland-3-0": 0, "wendland-3-1": 1, "wendland-3-3": 2, "wendland-3-2": 3}
# Pinned copies of the config table (bench.py --impl reference must not import
# the package, whose generators live in its own .so); checked against
# paper_1806_07884_b200/configs.py by tests/test_bench_contract.py.
CFG = {
    "cfg1": dict(dim=2, n=100_000, m=1_000, kernel="wendland-3-1", per_support=30,
                 desc="2D Halton N=1e5, h=Franke; M=1e3 Halton centres; phi31, ~30 centres/support"),
    "cfg2": dict(dim=2, n=1_000_000, m=10_000, kernel="wendland-3-1", per_support=50,
                 desc="2D uniform N=1e6, h=sin4x cos4y + N(0,0.01); M=1e4 on a 100x100 grid; phi31, ~50/support"),
    "cfg3": dict(dim=3, n=4_000_000, m=50_000, kernel="wendland-3-2", per_support=60,
                 desc="3D uniform N=4e6, h=exp(-|x-.5|^2/.1)+.5 sin6z; M=5e4 Halton; phi32, ~60/support"),
    "cfg4": dict(dim=2, n=20_000_000, m=100_000, kernel="wendland-3-1", per_support=40,
                 desc="2D Gaussian mixture N=2e7 (+5% uniform floor), h=6-octave fBm; M=1e5 Halton; phi31, ~40/support"),
    "cfg5": dict(dim=2, n=200_000_000, m=1_000_000, kernel="wendland-3-1", per_support=40,
                 desc="2D Halton N=2e8, h=Franke+N(0,0.001); M=1e6 on a 1000x1000 grid; phi31, ~40/support"),
}


def alpha_of(name: str) -> float:
    import math
    c = CFG[name]
    if c["dim"] == 2:
        r = math.sqrt(c["per_support"] / (math.pi * c["m"]))
    else:
        r = (c["per_support"] / (c["m"] * 4.0 * math.pi / 3.0)) ** (1.0 / 3.0)
    return 1.0 / r


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default=DEFAULT_CONFIG, choices=sorted(CFG))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=None, help="timed e2e fits (default: --steps)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--tile-div", type=float, default=None, help="sub-tile edge = radius / this")
    ap.add_argument("--super-factor", type=int, default=None, help="super-tile = this^dim sub-tiles")
    return ap.parse_args()


def dist_env():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def workload(name: str) -> dict:
    """The workload description, identical for both arms and every N."""
    c = CFG[name]
    return {"workload": f"{name}: {c['desc']}", "n_points": c["n"], "m_centres": c["m"], "dim": c["dim"],
            "kernel": c["kernel"], "alpha": alpha_of(name),
            "l2": "inputs (>= 1.6 GB at cfg3-5) exceed L2; a 256 MiB device write flushes L2 before every step "
                  "(outside the step events)"}


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi sampling during the timed region (recipe's clocks line)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self) -> dict:
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = max(mx, float(parts[2]))
            except ValueError:
                continue
            for n, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------ reference window sample
def _np_noise(seed: int, pos: np.ndarray, sigma: float) -> np.ndarray:
    """sigma * N(0,1) at array positions `pos`: restates the counter-based
    normal01 of csrc/datagen.cpp (splitmix64, Box-Muller) in numpy, so the
    reference arm needs no library of this package (libm ulp differences only)."""
    M = np.uint64(0xFFFFFFFFFFFFFFFF)

    def mix(x):
        x = (x + np.uint64(0x9E3779B97F4A7C15)) & M
        x = ((x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)) & M
        x = ((x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)) & M
        return x ^ (x >> np.uint64(31))

    def uni(i):
        k = mix(np.uint64(seed) ^ mix((np.uint64(0x6E6F726D) * np.uint64(0x632BE59BD9B4E019)) + i))
        return (k >> np.uint64(11)).astype(np.float64) * 2.0 ** -53

    with np.errstate(over="ignore"):
        i = pos.astype(np.uint64)
        u1 = 1.0 - uni(np.uint64(2) * i)
        u2 = uni(np.uint64(2) * i + np.uint64(1))
    return sigma * (np.sqrt(-2.0 * np.log(u1)) * np.cos(6.283185307179586 * u2))


def reference_window(name: str):
    """A spatial window of the config's workload built with the reference's
    own generators (oracle/_ref): every window point and all centres within
    the support radius of the window, so each point sees its full support.
    Halton configs: W = [0, 2^-a) x [0, 3^-b) holds exactly the sequence
    indices that are multiples of 2^a 3^b.  Returns (xy, h, refs, description)."""
    from oracle import pyoracle as po
    c = CFG[name]
    alpha = alpha_of(name)
    r = 1.0 / alpha
    if name not in ("cfg1", "cfg5"):
        raise NotImplementedError(name)
    a, b = (4, 3) if name == "cfg5" else (1, 1)
    stride = 2 ** a * 3 ** b
    idx = np.arange(stride, c["n"] + 1, stride, dtype=np.uint64)
    xy = po.ref_halton_at(idx, 2)
    h = po.ref_franke(xy)
    if name == "cfg5":
        h = h + _np_noise(5 * 1000 + 1, idx - np.uint64(1), 0.001)
        refs = po.ref_grid_refs(1000, 1000)
    else:
        refs = po.ref_halton_at(np.arange(1, c["m"] + 1, dtype=np.uint64), 2)
    wx, wy = 2.0 ** -a, 3.0 ** -b
    sel = (refs[:, 0] > -r) & (refs[:, 0] < wx + r) & (refs[:, 1] > -r) & (refs[:, 1] < wy + r)
    refs = np.ascontiguousarray(refs[sel])
    desc = (f"spatial window [0, 2^-{a}) x [0, 3^-{b}) of {name}: its {len(h)} points (Halton indices "
            f"multiple of {stride}) and the {len(refs)} centres within the support radius of it")
    return xy, h, refs, desc


def reference_fit(xy, h, refs, family: int, alpha: float, threads: int) -> dict:
    """The reference's fit (solver.cpp:401-478) on one sample: its PointIndex +
    assemble_submatrix + transpose_matvec + gram_self (oracle/_ref, single
    block, dense B -- solver.cpp:131-236) on `threads` point shards in
    parallel, partial systems summed, then solve_weights' ridge-laddered
    Cholesky (solver.cpp:289-330) with OpenBLAS dpotrf standing in for Eigen."""
    import concurrent.futures as cf

    import scipy.linalg as sl

    from oracle import pyoracle as po
    m = len(refs)
    shards = np.array_split(np.arange(len(h)), threads)
    t0 = time.perf_counter()
    with cf.ThreadPoolExecutor(max_workers=threads) as ex:  # ctypes releases the GIL
        parts = list(ex.map(lambda ix: po.ref_build_normal_system(xy[ix], h[ix], refs, family, alpha), shards))
    b = parts[0]["b"]
    rhs = parts[0]["rhs"].copy()
    for p in parts[1:]:
        b += p["b"]
        rhs += p["rhs"]
    t_build = time.perf_counter() - t0
    mean_diag = np.trace(b) / m
    lam_used = None
    for lam in (0.0, 1e-10, 1e-9, 1e-8, 1e-7, 1e-6):
        try:
            work = b + lam * mean_diag * np.eye(m) if lam > 0 else b
            c = sl.cho_solve(sl.cho_factor(work, lower=True, check_finite=False), rhs, check_finite=False)
            lam_used = lam
            break
        except np.linalg.LinAlgError:
            continue
    t_fit = time.perf_counter() - t0
    return {"build_s": t_build, "fit_s": t_fit, "ridge_lambda": lam_used, "c": c if lam_used is not None else None,
            "design_nnz": int(sum(p["design_nnz"] for p in parts))}


def host_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


# ------------------------------------------------------------- reference arm
def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:  # under torchrun only rank 0 runs the CPU reference
        return
    name = args.config
    c = CFG[name]
    fam = FAMILY[c["kernel"]]
    alpha = alpha_of(name)
    threads = host_threads()
    if name in ("cfg1", "cfg5"):
        xy, h, refs, desc = reference_window(name)
        kind = "reference"

        def step():
            return reference_fit(xy, h, refs, fam, alpha, threads)
        what = ("reference fit: kd-tree + assemble_submatrix + transpose_matvec + gram_self (oracle/_ref, one "
                "instance per host thread on point shards, partial systems summed) + ridge-laddered dense "
                "Cholesky (OpenBLAS dpotrf standing in for Eigen's LLT)")
    else:
        # configs the reference cannot hold (3-D, or dense M x M beyond host RAM): the
        # C restatement (oracle/rbf_oracle.c, threaded by output rows) + a sparse direct solve
        from oracle import pyoracle as po
        from paper_1806_07884_b200 import configs  # input generation only (outside the timed step)
        n = min(c["n"], 1_000_000)
        xy, h = configs.points(name, n=n)
        refs = configs.centres(name)
        desc = f"first {n} points of {name} with all {c['m']} centres"
        kind = "port"

        def step():
            import scipy.sparse as sp
            import scipy.sparse.linalg as spl
            t0 = time.perf_counter()
            rp, cols = po.pattern(refs, alpha)
            v, rhs, _ = po.assemble(xy, h, refs, fam, alpha, rp, cols)
            t_build = time.perf_counter() - t0
            rows = np.repeat(np.arange(len(refs)), np.diff(rp.astype(np.int64)))
            U = sp.csr_matrix((v, (rows, cols.astype(np.int64))), shape=(len(refs),) * 2)
            spl.spsolve((U + sp.triu(U, 1).T).tocsc(), rhs)
            return {"build_s": t_build, "fit_s": time.perf_counter() - t0}
        what = "C restatement (oracle/rbf_oracle.c) assembly + scipy sparse direct solve"
    for _ in range(args.warmup):
        step()
    res = [step() for _ in range(args.steps)]
    t = sum(r["fit_s"] for r in res) / len(res)
    tb = sum(r["build_s"] for r in res) / len(res)
    n = len(h)
    value = n / t
    sample = f"{desc}; {what}; {threads} host threads; per step build {tb:.3f} s, fit {t:.3f} s"
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload(name), "impl": "reference",
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": kind, "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "reference_assembly_points_per_s": n / tb,
            "ridge_lambda": res[-1].get("ridge_lambda")}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ our arm
def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_1806_07884_b200 import api, configs, distributed

    rank, world, local = dist_env()
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    # a real (non-legacy) stream shared by torch and the engine: the step events
    # and the NCCL all-reduce are ordered with the engine's kernels
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)

    name = args.config
    cfg = configs.CONFIGS[name]
    xy, h = configs.slab_points(name, rank, world)
    refs = configs.centres(name)
    kernel = api.KernelSpec(cfg.kernel, cfg.alpha)
    eng = api.Engine(local, stream=stream.cuda_stream)
    if args.tile_div:
        eng.set_tile_divisor(args.tile_div)
    if args.super_factor:
        eng.set_super_factor(args.super_factor)
    eng.set_centres(refs, kernel)
    info = eng.pattern_info()
    d_xy = torch.from_numpy(xy).cuda()
    d_h = torch.from_numpy(h).cuda()
    n = len(h)
    sys_t = distributed.system_tensor(eng)

    def step():
        eng.assemble_device(d_xy.data_ptr(), d_h.data_ptr(), n)
        if world > 1:
            dist.all_reduce(sys_t)

    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    lay = eng.layout_info()
    # algorithmic work of this rank's step (outside timing): sum_k F + k(k+1) + 2k
    sum_k, sum_k2 = _ncounts(eng, xy)
    flops_step = sum_k2 + (F_PHI[cfg.dim] + 3) * sum_k
    bytes_step = n * (cfg.dim + 1) * 8 + info["nnz_upper"] * 12 + cfg.m * 8
    fp64_peak = _fp64_peak(eng)

    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    tile_ms, bin_ms = [], []
    launches0 = eng.launch_count
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clocks:
        for k in range(args.steps):
            flush.fill_(float(k))
            starts[k].record(stream)
            step()
            ends[k].record(stream)
            b, t = _asm_times(eng)  # events on the engine stream, read after the step
            bin_ms.append(b)
            tile_ms.append(t)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches = eng.launch_count - launches0
    total_ms = sum(s.elapsed_time(e) for s, e in zip(starts, ends))
    total_ms = _max_over_ranks(total_ms, world)
    ms_per_step = total_ms / args.steps
    n_total = _sum_over_ranks(n, world)
    value = n_total / (ms_per_step * 1e-3)

    e2e = None if args.no_e2e else _e2e(xy, h, refs, kernel, cfg, world, rank, local, args, stream)

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    t_tile = statistics.median(tile_ms) * 1e-3
    achieved = flops_step / t_tile / 1e12
    roof = {"bound": "fp64", "achieved": achieved, "peak": fp64_peak, "unit": "TFLOP/s",
            "frac": achieved / fp64_peak, "traffic": _traffic(name),
            "kernel": "assemble_warp_kernel (persistent one-warp workers: phi into DMMA fragments, register "
                      "SYRK per sub-tile, warp-private super-tile accumulator, slot-map flush)",
            "peak_source": "measured live: rbg_fp64_peak DFMA microbenchmark (MEASURED_PEAKS.json has no fp64)",
            "algorithmic_flops_per_launch": flops_step, "kernel_ms": t_tile * 1e3,
            "kernel_share_of_step": t_tile * 1e3 / ms_per_step,
            "bin_ms": statistics.median(bin_ms),
            "hbm": {"algorithmic_bytes": bytes_step, "achieved_gbs": bytes_step / t_tile / 1e9,
                    "peak_gbs": _hbm_peak(), "frac": bytes_step / t_tile / 1e9 / _hbm_peak()}}
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(name)
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload(name),
            "parallelism": (f"{world} ranks x equal-count spatial slabs, one NCCL all-reduce of "
                            f"[values|rhs|hits] per step" if world > 1 else "1 GPU"),
            "clocks": clocks.summary(), "roofline": roof, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": launches,
            "detail": {"points_this_rank": n, "nnz_upper": info["nnz_upper"], "setup_ms": info["setup_ms"],
                       "sum_k": sum_k, "sum_k2": sum_k2,
                       "layout": {k: (round(v, 2) if isinstance(v, float) else v) for k, v in lay.items()}}}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def _max_over_ranks(v: float, world: int) -> float:
    if world == 1:
        return v
    import torch
    import torch.distributed as dist
    t = torch.tensor([v], device="cuda", dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def _sum_over_ranks(v: int, world: int) -> int:
    if world == 1:
        return v
    import torch
    import torch.distributed as dist
    t = torch.tensor([v], device="cuda", dtype=torch.int64)
    dist.all_reduce(t)
    return int(t.item())


def _e2e(xy, h, refs, kernel, cfg, world, rank, local, args, stream):
    """The public fit from pageable host arrays, a fresh context per step."""
    import torch
    import torch.distributed as dist

    from paper_1806_07884_b200 import api, distributed
    steps = args.e2e_steps or args.steps

    def fit_once():
        t0 = time.perf_counter()
        if world == 1:
            model, rep = api.fit(xy, h, refs, kernel, engine=api.Engine(local))
            c = model.weights
        else:  # strong scaling: slab assembly, all-reduce on the engine stream, every rank solves
            rep = api.FitReport()
            with api.Engine(local, stream=stream.cuda_stream) as e:
                e.set_centres(refs, kernel)
                e.assemble(xy, h)
                distributed.allreduce_system(e)
                c, d = e.solve()
                rep.iterations, rep.solve_ms = d["iterations"], d["solve_ms"]
        return time.perf_counter() - t0, c, rep

    fit_once()
    if world > 1:
        dist.barrier()
    times, rep = [], None
    for _ in range(steps):
        dt, c, rep = fit_once()
        times.append(dt)
    dt = _max_over_ranks(sum(times) / len(times), world)
    n_total = _sum_over_ranks(len(h), world)
    return {"value": n_total / dt, "unit": UNIT, "ms_per_step": dt * 1e3, "steps": steps,
            "ms_min": min(times) * 1e3, "ms_median": statistics.median(times) * 1e3, "ms_max": max(times) * 1e3,
            "h2d_bytes_per_step": int(len(h) * (cfg.dim + 1) * 8 + refs.size * 8),
            "d2h_bytes_per_step": int(cfg.m * 8 + (cfg.m * 8 if world == 1 else 0)),
            "api": ("api.fit -> rbg_create, rbg_set_centres, rbg_assemble (pageable host arrays, validated), "
                    "rbg_get_system (hit counts), rbg_solve (c to the host)" if world == 1 else
                    "rbg_create, rbg_set_centres, rbg_assemble (host slab), NCCL all-reduce, rbg_solve"),
            "fit": {"setup_ms": getattr(rep, "setup_ms", None), "solve_ms": rep.solve_ms,
                    "iterations": rep.iterations, "ridge_lambda": getattr(rep, "ridge_lambda", None)}}


def cpu_baseline(name: str) -> dict | None:
    """The reference's CPU fit on the same bounded window the reference arm
    uses (kind 'reference'), or the C restatement where the reference cannot
    run the config (kind 'port')."""
    c = CFG[name]
    threads = host_threads()
    fam = FAMILY[c["kernel"]]
    try:
        if name in ("cfg1", "cfg5"):
            xy, h, refs, desc = reference_window(name)
            reference_fit(xy, h, refs, fam, alpha_of(name), threads)  # warm
            r = reference_fit(xy, h, refs, fam, alpha_of(name), threads)
            return {"value": len(h) / r["build_s"], "unit": UNIT, "cores": threads, "kind": "reference",
                    "sample": f"{desc}; reference index + assemble_submatrix + gram_self on {threads} threads "
                              f"({r['build_s']:.3f} s); the whole reference fit incl. Cholesky "
                              f"{r['fit_s']:.3f} s = {len(h) / r['fit_s']:.4g} points/s"}
        from oracle import pyoracle as po
        from paper_1806_07884_b200 import configs
        n = min(c["n"], 1_000_000)
        xy, h = configs.points(name, n=n)
        refs = configs.centres(name)
        rp, cols = po.pattern(refs, alpha_of(name))
        t0 = time.perf_counter()
        po.assemble(xy, h, refs, fam, alpha_of(name), rp, cols)
        t = time.perf_counter() - t0
        return {"value": n / t, "unit": UNIT, "cores": threads, "kind": "port",
                "sample": f"first {n} points of {name}, all {c['m']} centres: C restatement "
                          f"(oracle/rbf_oracle.c, OpenMP by output rows), pattern excluded"}
    except Exception as e:  # the baseline is reported, never required
        return {"value": None, "unit": UNIT, "cores": threads, "kind": "reference", "sample": f"failed: {e}"}


def _ncounts(eng, xy):
    import ctypes as C

    from paper_1806_07884_b200 import _native
    a, b = C.c_uint64(), C.c_uint64()
    _native.check(_native.lib().rbg_support_counts(eng._ctx, xy.ctypes.data, len(xy), C.byref(a), C.byref(b)),
                  eng._ctx)
    return int(a.value), int(b.value)


def _fp64_peak(eng):
    import ctypes as C

    from paper_1806_07884_b200 import _native
    v = C.c_double()
    _native.check(_native.lib().rbg_fp64_peak(eng._ctx, C.byref(v)), eng._ctx)
    return v.value


def _asm_times(eng):
    import ctypes as C

    from paper_1806_07884_b200 import _native
    a, b = C.c_double(), C.c_double()
    _native.check(_native.lib().rbg_assembly_times(eng._ctx, C.byref(a), C.byref(b)), eng._ctx)
    return a.value, b.value


def _hbm_peak():
    try:
        return float(json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"])
    except Exception:
        return 6650.0  # B200_PROFILING.md fallback


def _traffic(name):
    p = ROOT / "profiles" / "traffic.json"
    try:
        return json.loads(p.read_text()).get(name)
    except Exception:
        return None


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
