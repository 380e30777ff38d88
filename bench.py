"""Benchmark: batched FP64 logm throughput (matrices/s) on B200, BASELINE.json's metric.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 4] [--impl ours|reference]

One *step* = one pass of the whole logm hot path (balance -> scaling loop with norm
estimation and DB square roots -> order selection -> graph polynomial -> 2^s rescale ->
unbalance) over one batch of matrices already resident in HBM.  Default workload is
BASELINE.json configs[3] (config 4: 256 float64 SPD 512x512 matrices, the largest
single-GPU configuration and north_star's n >= 512 roofline regime), strong scaling: the
256-matrix global batch is split by matrix across the ranks, no data-path collective, and
the result gather to rank 0 (NCCL) is inside the timed region.
Under torchrun each rank drives one GPU; timings are CUDA events on the launching
stream, the max over ranks is reported.  The L2 (126 MB) is flushed between timed steps
(256 MiB write) so small batches (config 2: 32 MiB) do not stay L2 resident.

``--impl reference`` times the reference algorithm's CPU implementation (the oracle port
of the reference primitives + restated driver, oracle/; the reference's own driver file
is missing) on all host cores over a bounded sample of the same workload.
"""
import argparse
import json
import math
import multiprocessing as mp
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "fp64 logm matrices/sec (batched, n=32..4096); achieved FP64 tensor TFLOP/s"
UNIT = "matrices/s"


def _peak_fp64():
    """Measured FP64 peak (tools/fp64_peak.cu): MEASURED_PEAKS.json has no FP64 entry."""
    p = os.path.join(ROOT, "profiles", "fp64_peak_r01.json")
    try:
        d = json.load(open(p))
        return float(d["dmma_tflops"]), "measured: profiles/fp64_peak_r01.json dmma_tflops (DMMA.8x8x4 microbenchmark)"
    except Exception:  # noqa: BLE001
        return 36.9, "fallback: round-1 DMMA microbenchmark"


def _peak_hbm():
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]), "MEASURED_PEAKS.json"
    except Exception:  # noqa: BLE001
        return 6650.0, "fallback B200_PROFILING.md"


def workload(cfg, batch=None, n=None, seed_offset=0):
    from paper_2401_10089_b200 import synth
    name, n0, b0 = synth.CONFIGS[cfg]
    n = n or n0
    batch = batch or b0
    seed = synth.SEEDS[cfg] + 7919 * seed_offset
    return synth.config(cfg, batch=batch, n=n, seed=seed), name


def flops_per_matrix(n, rec):
    """F = 2n^3 [sum_r (2 it_r - 1) + (k - 1) + 1(s = 0)] + 4 n^2 E."""
    s, its, k, E = int(rec["s"]), int(rec["db_iters"]), int(rec["k"]), int(rec["estimation_passes"])
    if int(rec["status"]) != 0:
        # failed matrices: the DB work actually done (every iteration after the first of a
        # root inverts both X and Y)
        return 2.0 * n ** 3 * max(2 * its - (s + 1), 0) + 4.0 * n * n * E
    return 2.0 * n ** 3 * ((2 * its - s) + (k - 1) + (1 if s == 0 else 0)) + 4.0 * n * n * E


def skipped_flops(n, rec):
    """Inversions of the reference's algorithm that the lazy-X^-1 order did not execute (a
    root's last DB iteration needs only Y^-1): reported beside the algorithmic count."""
    return 2.0 * n ** 3 * int(rec["inv_skipped"])


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled in the background (B200_PROFILING.md)."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                          "-lms", "50", "-i", str(self.index)], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:  # noqa: BLE001
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:  # noqa: BLE001
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        busy = [v for v in sm if v > 600] or sm
        return {"sm_mhz": statistics.median(busy) if busy else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------------------- CPU side

def _cpu_worker_init():
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    if ROOT not in sys.path:
        sys.path.insert(0, ROOT)


def _cpu_worker(chunk):
    from oracle import driver as D
    prims = D.default_prims()
    ok = 0
    for A in chunk:
        prims.margins = type(prims.margins)()
        _, rep = D.logm_status(A, prims)
        ok += rep["status"] == 0
    return ok


def _cpu_serial(As, cores):
    """Mode 1 of BASELINE.md section 2: serial over matrices, BLAS on all cores (a spawned
    child so OPENBLAS_NUM_THREADS takes effect)."""
    ctx = mp.get_context("spawn")
    os.environ["OPENBLAS_NUM_THREADS"] = str(cores)
    with ctx.Pool(1, initializer=_cpu_serial_init, initargs=(cores,)) as pool:
        pool.map(_cpu_worker, [As[:1]])
        t0 = time.perf_counter()
        pool.map(_cpu_worker, [As])
        return time.perf_counter() - t0


def _cpu_serial_init(cores):
    os.environ["OPENBLAS_NUM_THREADS"] = str(cores)
    if ROOT not in sys.path:
        sys.path.insert(0, ROOT)


def cpu_mode(n):
    """The faster of BASELINE.md's two modes for this size (measured on the B200 box's 16
    host cores: the pool wins up to n = 512 -- 6.3 vs 1.8 matrices/s at config 4 -- all-core
    BLAS is kept for n >= 2048, where one matrix per core would not fit the time budget)."""
    return "pool" if n <= 1024 else "serial"


def mode_text(n, cores):
    return (f"process pool x{cores}, OPENBLAS_NUM_THREADS=1" if cpu_mode(n) == "pool"
            else f"serial over matrices, OPENBLAS_NUM_THREADS={cores}")


def cpu_time(As, cores):
    """Time the oracle port over matrices As on `cores` host cores.  Returns wall seconds."""
    if cpu_mode(As.shape[-1]) == "serial":
        return _cpu_serial(As, cores)
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    ctx = mp.get_context("spawn")
    chunks = [c for c in np.array_split(As, max(1, min(len(As), cores * 4))) if len(c)]
    with ctx.Pool(cores, initializer=_cpu_worker_init) as pool:
        pool.map(_cpu_worker, [chunks[0][:1]] * cores)          # warm the workers
        t0 = time.perf_counter()
        pool.map(_cpu_worker, chunks)
        return time.perf_counter() - t0


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:  # noqa: BLE001
        return os.cpu_count() or 1


# ----------------------------------------------------------------------------- main

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="4")
    ap.add_argument("--batch", type=int, default=None, help="GLOBAL matrices (default: the config's)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-sample", type=int, default=None)
    ap.add_argument("--max-k", type=int, default=None,
                    help="LogmOptions.max_k (default 5: the reference's shipped schemes; 6..9 opt-in)")
    args = ap.parse_args()
    cfg = args.config if args.config in ("3b", "5b") else int(args.config)
    args.warmup = max(args.warmup, 3)

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        return run_reference(args, cfg, rank, world)

    import torch
    import torch.distributed as dist
    import paper_2401_10089_b200 as lp
    from paper_2401_10089_b200 import _lib, driver
    from paper_2401_10089_b200.multigpu import gather_tensor_to, shard_bounds

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    # strong scaling: the config's GLOBAL batch (config 4: 256 matrices) split by matrix
    # across the ranks; results gathered to rank 0 inside the timed region
    A_all, name = workload(cfg, batch=args.batch)
    Bg, n, _ = A_all.shape
    lo, hi = shard_bounds(Bg, world)[rank]
    A_np = np.ascontiguousarray(A_all[lo:hi])
    B = A_np.shape[0]
    A = torch.from_numpy(A_np).to(dev)
    opts = lp.LogmOptions(raise_on_error=False) if args.max_k is None else \
        lp.LogmOptions(raise_on_error=False, max_k=args.max_k)
    stream = torch.cuda.current_stream(dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.int32, device=dev)

    def step():
        L, rep, ws = driver.run_device(A, opts, stream)
        Lg = gather_tensor_to(L, rank, world, Bg)          # result gather (NCCL), no-op at N = 1
        return L, rep, Lg

    for _ in range(args.warmup):
        L, rep, _ = step()
    torch.cuda.synchronize()
    reps = rep.cpu().numpy().view(_lib.REPORT_DTYPE)[:B]

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    times = []
    launches0 = _lib.launch_count()
    with ClockSampler(local_rank) as clk:
        barrier()
        for _ in range(args.steps):
            flush.zero_()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            step()
            e1.record(stream)
            times.append((e0, e1))
        barrier()
    launches = _lib.launch_count() - launches0
    kernel_ms = [a.elapsed_time(b) for a, b in times]
    t = torch.tensor([sum(kernel_ms)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    value = Bg * args.steps / (total_ms * 1e-3)

    # roofline: algorithmic FLOPs of one step (all ranks' matrices) / step time (max over ranks)
    Fl = torch.tensor([sum(flops_per_matrix(n, r) for r in reps), sum(skipped_flops(n, r) for r in reps)],
                      dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(Fl)
    F, F_skip = float(Fl[0].item()), float(Fl[1].item())
    peak, peak_src = _peak_fp64()
    step_s = ms_per_step * 1e-3
    achieved = F / step_s / 1e12
    hbm_peak, hbm_src = _peak_hbm()
    alg_bytes = Bg * (16.0 * n * n + _lib.REPORT_DTYPE.itemsize)
    traffic, kernel_share = None, None
    try:
        tr = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic_r02.json")))
        ent = tr.get(str(args.config), {})
        traffic = ent.get("dram_bytes_per_step")
        kernel_share = ent.get("kernel_share")
    except Exception:  # noqa: BLE001
        pass

    # end-to-end through the public API with host (pinned) buffers: H2D of this rank's inputs,
    # the whole logm, D2H of L and the reports, every step
    e2e_value = None
    if not args.no_e2e:
        A_host = torch.from_numpy(A_np).pin_memory()
        L_host = torch.empty_like(A_host).pin_memory()      # the caller's reusable output buffer
        for _ in range(2):
            lp.logm_batched(A_host, opts, out=L_host)
        e2e_times = []
        for _ in range(max(3, min(args.steps, 10))):
            barrier()
            t0 = time.perf_counter()
            lp.logm_batched(A_host, opts, out=L_host)
            e2e_times.append(time.perf_counter() - t0)
        te = torch.tensor([sum(e2e_times) / len(e2e_times)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e_value = Bg / float(te.item())

    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return

    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        cores = host_cores()
        sample = args.cpu_sample or (B if n <= 64 else min(B, 16 * cores) if n <= 256 else
                                     min(B, 2 * cores) if n <= 1024 else 1)
        secs = cpu_time(A_np[:sample], cores)
        cpu = {"value": sample / secs, "unit": UNIT, "cores": cores, "kind": "port",
               "sample": f"first {sample} of the {B} config-{args.config} matrices, oracle port "
                         f"(oracle/driver.py over numpy/scipy/OpenBLAS), {mode_text(n, cores)}, "
                         f"{secs:.2f} s wall"}

    status_counts = {int(s): int(c) for s, c in zip(*np.unique(reps["status"], return_counts=True))}
    engine = "F (fused, 1 CTA/matrix)" if n <= 64 else "G (batched grid, device-driven)"
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded numpy generator, synth.py)",
        "config": {"workload": f"config{args.config}:{name}", "n": n, "global_batch": Bg,
                   "batch_per_gpu": B, "parallelism": f"batch-sharded x{world} (no collective; result gather "
                                                      f"to rank 0 inside the timed region)",
                   "l2": "flushed between timed steps (256 MiB write)", "engine": engine,
                   "max_k": opts.max_k},
        "achieved_tflops": achieved,
        "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                     "kernel": ("logm_fused_kernel<32>" if n <= 32 else "logm_fused_kernel<64>") if n <= 64
                     else "whole Engine-G logm step (achieved = step algorithmic FLOPs / step time)",
                     "kernel_share": kernel_share,
                     "alg_flops_per_step": F,
                     "executed": {"flops_per_step": F - F_skip, "tflops": (F - F_skip) / step_s / 1e12,
                                  "frac": (F - F_skip) / step_s / 1e12 / peak,
                                  "note": "algorithmic count minus the DB X-inversions the lazy order skips "
                                          "(report inv_skipped); achieved/frac above use the SURVEY 8(d) "
                                          "algorithmic count of the reference algorithm"},
                     "hbm": {"achieved_gbs": alg_bytes / step_s / 1e9, "peak_gbs": hbm_peak,
                             "frac": alg_bytes / step_s / 1e9 / hbm_peak, "alg_bytes_per_step": alg_bytes,
                             "peak_source": hbm_src}},
        "cpu_baseline": cpu,
        "e2e": None if e2e_value is None else
        {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(B * n * n * 8),
         "d2h_bytes_per_step": int(B * n * n * 8 + B * _lib.REPORT_DTYPE.itemsize)},
        "gpu_launches": launches,
        "clocks": clk.summary(),
        "report_summary": {"status_counts": status_counts, "s_mean": float(reps["s"].mean()),
                           "k_mean": float(reps["k"].mean()), "db_iters_mean": float(reps["db_iters"].mean()),
                           "estimation_passes_mean": float(reps["estimation_passes"].mean())},
    }
    print(json.dumps(line))
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def run_reference(args, cfg, rank, world):
    """The reference algorithm's CPU implementation on all host cores (rank 0 only)."""
    if rank != 0:
        return
    A_np, name = workload(cfg, batch=args.batch)
    B, n, _ = A_np.shape
    cores = host_cores()
    sample = args.cpu_sample or (256 if n <= 64 else min(B, 4 * cores) if n <= 256 else
                                 min(B, cores) if n <= 1024 else 1)
    sample = min(sample, B)
    # one persistent pool (or one all-core-BLAS child) for the whole run; warm-up steps first
    pool_mode = cpu_mode(n) == "pool"
    os.environ["OPENBLAS_NUM_THREADS"] = "1" if pool_mode else str(cores)
    ctx = mp.get_context("spawn")
    procs = cores if pool_mode else 1
    init, iargs = (_cpu_worker_init, ()) if pool_mode else (_cpu_serial_init, (cores,))
    secs = []
    with ctx.Pool(procs, initializer=init, initargs=iargs) as pool:
        def one_step(chunk):
            parts = [c for c in np.array_split(chunk, max(1, min(len(chunk), procs * 4))) if len(c)]
            t0 = time.perf_counter()
            pool.map(_cpu_worker, parts, chunksize=1)
            return time.perf_counter() - t0
        for _ in range(min(args.warmup, 1)):
            one_step(A_np[:min(sample, procs)])
        for s in range(args.steps):
            lo = (s * sample) % B
            chunk = A_np[lo:lo + sample] if lo + sample <= B else A_np[:sample]
            secs.append(one_step(chunk))
    total = sum(secs)
    value = sample * args.steps / total
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": total / args.steps * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded numpy generator, synth.py)",
        "config": {"workload": f"config{args.config}:{name}", "n": n, "global_batch": B},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": f"{sample} matrices of config {args.config} per step, oracle port "
                                   f"(oracle/driver.py: restated driver over the numpy/scipy restatement of the "
                                   f"reference primitives), {mode_text(n, cores)}"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


if __name__ == "__main__":
    main()
