#!/usr/bin/env python
"""Benchmark of the CS-RBF normal-equation hot path (BASELINE.json metric:
A^T A assembly points/s, fit time, roofline fraction).

One step = one pass of the hot path over one batch: bin the batch's points
into the centre tiles and assemble A^T A and A^T h (+ the NCCL allreduce of the
partial systems when N > 1).  The centre set / symbolic pattern depends only on
the centres and is built once before timing (reported as setup_ms).

  python bench.py [--gpus N --steps K --warmup W] [--config cfg2] [--impl reference]

N > 1 runs under torchrun (one rank per GPU, NCCL).  Weak scaling: every rank
assembles an independent full-size draw of the config's point distribution
against the shared centres; value = all ranks' points / max-over-ranks time.
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
F_PHI = {2: 14, 3: 20}  # flops per phi evaluation incl. distance
REF_SAMPLE = 250_000  # reference arm: points per CPU step (bounded sample)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-fit", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--tile-div", type=float, default=None, help="sub-tile edge = radius / this")
    ap.add_argument("--super-factor", type=int, default=None, help="super-tile = this^dim sub-tiles")
    return ap.parse_args()


def dist_env():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def workload(cfg) -> dict:
    return {"workload": f"{cfg.name}: {cfg.description}", "n_points_per_rank": cfg.n, "m_centres": cfg.m,
            "dim": cfg.dim, "kernel": cfg.kernel, "alpha": cfg.alpha,
            "l2": "flushed between timed steps (256 MiB device write outside the step events)"}


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


# ------------------------------------------------------------ cpu baseline
def cpu_baseline(cfg, xy, h, refs, samples: int = 3) -> dict:
    """The reference's own CPU path (oracle/_ref, compiled from the reference
    sources) on a bounded sample, 1 thread (the reference is single-threaded).
    Falls back to our C restatement when the reference could not run here."""
    from oracle import pyoracle as po

    n = min(REF_SAMPLE, len(h))
    fam = {"wendland-3-0": 0, "wendland-3-1": 1, "wendland-3-3": 2, "wendland-3-2": 3}[cfg.kernel]
    if po.ref_available() and cfg.dim == 2 and cfg.m <= 20_000 and fam <= 2:
        times = []
        for _ in range(samples):
            sec, _dn = po.ref_bench_step(xy[:n], h[:n], refs, fam, cfg.alpha)
            times.append(sec)
        t = statistics.median(times)
        return {"value": n / t, "unit": UNIT, "cores": 1, "kind": "reference",
                "sample": f"first {n} points of {cfg.name} with all {cfg.m} centres; reference "
                          f"kd-tree + assemble_submatrix + transpose_matvec + gram_self "
                          f"(single block), median of {samples}, {t:.2f} s each"}
    # restatement (sparse, point-ascending) for configs the reference cannot hold
    n = min(n, 100_000)
    t0 = time.perf_counter()
    rp, cols = po.pattern(refs, cfg.alpha)
    t_pat = time.perf_counter() - t0
    times = []
    for _ in range(samples):
        t0 = time.perf_counter()
        po.assemble(xy[:n], h[:n], refs, fam, cfg.alpha, rp, cols)
        times.append(time.perf_counter() - t0)
    t = statistics.median(times)
    return {"value": n / t, "unit": UNIT, "cores": 1, "kind": "port",
            "sample": f"first {n} points of {cfg.name}, all {cfg.m} centres; C restatement "
                      f"(oracle/rbf_oracle.c), pattern {t_pat:.2f} s excluded, median of {samples}"}


# ------------------------------------------------------------- reference arm
def run_reference(args, cfg):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from oracle import pyoracle as po
    from paper_1806_07884_b200 import configs

    xy, h = configs.points(cfg.name, n=min(REF_SAMPLE, cfg.n))
    refs = configs.centres(cfg.name)
    fam = {"wendland-3-0": 0, "wendland-3-1": 1, "wendland-3-3": 2, "wendland-3-2": 3}[cfg.kernel]
    n = len(h)
    threads = 1
    if po.ref_available() and cfg.dim == 2 and cfg.m <= 20_000 and fam <= 2:
        kind = "reference"
        # The reference is single-threaded; to give it every host core we run
        # one independent reference instance per core on its own shard of the
        # sample (partial normal systems add, exactly like the GPU point shards).
        # Each instance holds a dense M x M block, so the count is also capped
        # by host memory.
        import concurrent.futures as cf
        try:
            import psutil
            avail = psutil.virtual_memory().available
        except Exception:
            avail = 16 << 30
        per_inst = 3 * cfg.m * cfg.m * 8 + (256 << 20)
        threads = max(1, min(os.cpu_count() or 1, 64, int(0.6 * avail // per_inst), n // 2000))
        shards = np.array_split(np.arange(n), threads)

        def step():
            t0 = time.perf_counter()
            with cf.ThreadPoolExecutor(max_workers=threads) as ex:  # ctypes releases the GIL
                list(ex.map(lambda ix: po.ref_bench_step(xy[ix], h[ix], refs, fam, cfg.alpha), shards))
            return time.perf_counter() - t0
        sample = (f"first {n} points of {cfg.name}, all {cfg.m} centres: reference kd-tree + "
                  f"assemble_submatrix + transpose_matvec + gram_self, single block, {threads} independent "
                  f"reference instances (one per host thread) on point shards")
    else:
        kind = "port"
        rp, cols = po.pattern(refs, cfg.alpha)
        n = min(n, 100_000)

        def step():
            t0 = time.perf_counter()
            po.assemble(xy[:n], h[:n], refs, fam, cfg.alpha, rp, cols)
            return time.perf_counter() - t0
        sample = f"first {n} points of {cfg.name}: C restatement (reference cannot hold this config)"
    for _ in range(args.warmup):
        step()
    times = [step() for _ in range(args.steps)]
    t = sum(times) / len(times)
    value = n / t
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload(cfg), "impl": "reference",
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": kind, "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ our arm
def run_ours(args, cfg):
    import torch
    import torch.distributed as dist

    from paper_1806_07884_b200 import _native, api, configs, distributed

    rank, world, local = dist_env()
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    # a real (non-legacy) stream shared by torch and the engine, so the step
    # events and NCCL are ordered with the engine's kernels
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)

    xy, h = configs.points(cfg.name, seed_offset=rank)
    refs = configs.centres(cfg.name)
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
    # algorithmic work of one step on this rank (outside timing)
    sum_k, sum_k2 = _ncounts(eng, xy)
    flops_step = sum_k2 + (F_PHI[cfg.dim] + 3) * sum_k  # sum k F + k(k+1) + 2k
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
            if world == 1:
                b, t = _asm_times(eng)
                bin_ms.append(b)
                tile_ms.append(t)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches = eng.launch_count - launches0
    total_ms = sum(s.elapsed_time(e) for s, e in zip(starts, ends))
    if world > 1:
        t = torch.tensor([total_ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    value = world * n / (ms_per_step * 1e-3)

    # e2e: public C-ABI call from pinned host buffers, result read back each step
    e2e = _e2e(eng, xy, h, info, cfg, world, args)

    fit = None if args.no_fit or rank != 0 else _fit_once(eng, xy, h)

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    roof = None
    if tile_ms:
        t_tile = statistics.median(tile_ms) * 1e-3
        achieved = flops_step / t_tile / 1e12
        roof = {"bound": "fp64", "achieved": achieved, "peak": fp64_peak, "unit": "TFLOP/s",
                "frac": achieved / fp64_peak, "traffic": _traffic(cfg.name),
                "kernel": "assemble_warp_kernel (persistent one-warp workers: phi into DMMA fragments, register SYRK per sub-tile, warp-private super-tile accumulator, slot-map flush)",
                "peak_source": "measured live: rbg_fp64_peak DFMA microbenchmark (MEASURED_PEAKS.json has no fp64)",
                "algorithmic_flops_per_launch": flops_step, "tile_ms": t_tile * 1e3,
                "bin_ms": statistics.median(bin_ms),
                "hbm": {"algorithmic_bytes": bytes_step, "achieved_gbs": bytes_step / t_tile / 1e9,
                        "peak_gbs": _hbm_peak(), "frac": bytes_step / t_tile / 1e9 / _hbm_peak()}}
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(cfg, xy, h, refs)
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {**workload(cfg), "parallelism": f"dp{world} (point shards, NCCL allreduce)",
                       "nnz_upper": info["nnz_upper"], "n_tiles": info["n_tiles"],
                       "setup_ms": info["setup_ms"], "sum_k": sum_k, "sum_k2": sum_k2,
                       "layout": {"sub_div": lay["sub_div"], "super_factor": lay["super_factor"],
                                  "n_super": lay["n_super"], "n_buckets": lay["n_buckets"],
                                  "n_fallback": lay["n_fallback"],
                                  "mean_super_centres": round(lay["mean_super_centres"], 2),
                                  "mean_sub_centres": round(lay["mean_sub_centres"], 2),
                                  "max_super_centres": lay["max_super_centres"],
                                  "max_sub_centres": lay["max_sub_centres"], "build_ms": round(lay["build_ms"], 2)}},
            "clocks": clocks.summary(), "roofline": roof, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": launches, "fit": fit}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


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


def _e2e(eng, xy, h, info, cfg, world, args):
    import ctypes as C

    import torch
    import torch.distributed as dist

    from paper_1806_07884_b200 import _native, distributed
    L = _native.lib()
    n = len(h)
    p_xy = torch.from_numpy(xy).pin_memory()
    p_h = torch.from_numpy(h).pin_memory()
    nnz, m = info["nnz_upper"], cfg.m
    o_v = torch.empty(nnz, dtype=torch.float64).pin_memory()
    o_r = torch.empty(m, dtype=torch.float64).pin_memory()
    o_hits = torch.empty(m, dtype=torch.float64).pin_memory()
    dn = C.c_uint64()
    sys_t = distributed.system_tensor(eng) if world > 1 else None
    steps = args.e2e_steps or args.steps

    def one():
        eng.assemble_ptr(p_xy.data_ptr(), p_h.data_ptr(), n)
        if world > 1:
            dist.all_reduce(sys_t)
        _native.check(L.rbg_get_system(eng._ctx, o_v.data_ptr(), o_r.data_ptr(), o_hits.data_ptr(),
                                       C.byref(dn)), eng._ctx)

    for _ in range(2):
        one()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(steps):
        one()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / steps
    if world > 1:
        t = torch.tensor([dt], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dt = float(t.item())
    return {"value": world * n / dt, "unit": UNIT, "ms_per_step": dt * 1e3,
            "h2d_bytes_per_step": n * (cfg.dim + 1) * 8, "d2h_bytes_per_step": (nnz + 2 * m) * 8,
            "api": "rbg_assemble (host pinned in) + rbg_get_system (host out)"}


def _fit_once(eng, xy, h):
    t0 = time.perf_counter()
    eng.assemble(xy, h, validate=True)
    eng.synchronize()
    t_asm = time.perf_counter() - t0
    c, diag = eng.solve()
    t1 = time.perf_counter()
    rep = eng.error_report(c, xy, h)
    t_err = time.perf_counter() - t1
    return {"assembly_s": t_asm, "solve_s": diag["solve_ms"] * 1e-3, "iterations": diag["iterations"],
            "rel_residual": diag["rel_residual"], "ridge_lambda": diag["ridge_lambda"],
            "eval_error_s": t_err, "fit_s": t_asm + diag["solve_ms"] * 1e-3,
            "mae": rep["mean_absolute_error"], "rms": rep["rms_error"], "max_abs": rep["max_abs_error"]}


def main():
    args = parse()
    from paper_1806_07884_b200 import configs

    cfg = configs.CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, cfg)
    else:
        run_ours(args, cfg)


if __name__ == "__main__":
    main()
