#!/usr/bin/env python3
"""Benchmark of the hot path (BASELINE.json metric "Winograd conv effective TFLOP/s
(direct-FLOP equiv) and c-sweep tiles/s at 1/2/4/8").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl native|reference]
    torchrun --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N ...

A STEP is the whole configs[1] job: four sweeps
(1D / 2D F(4,3) x uniform / normal tiles) of 4096 log-spaced c over 100,000 shared random
tiles each, every output scored against fp64 direct correlation, candidates sharded over
the ranks, statistics all-reduced (NCCL).  `value` = tile-evaluations per second of the
whole job (candidates x tiles, all four sweeps) -- strong scaling: the job is fixed, ranks
split the candidates.  The configs[2] layer (a3-a7, F(6x6,3x3), N=32 C=K=256 56x56) is
measured on rank 0 beside it and reported under "layer" (effective direct-equivalent
TFLOP/s), unscored and scored.

Timing: W untimed warm-up steps; K timed steps, each bracketed by CUDA events on the
launching stream, the L2 flushed (512 MB write) between steps outside the events;
barrier + synchronize around the timed region; max over ranks.  Clocks are sampled with
NVML during the timed region.  `e2e` repeats the job through the same C-ABI call with the
tiles copied H2D from pinned host memory (on a copy stream, each sweep waiting for its own
tiles, so later sweeps' copies overlap earlier sweeps' kernels) and the statistics copied
back D2H inside the timed region.  `cpu_baseline` / `--impl reference` time the oracle (oracle/, plain C,
OpenMP) on the host cores on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = "Winograd conv effective TFLOP/s (direct-FLOP equiv) and c-sweep tiles/s at 1/2/4/8"
N_C = 4096
N_TILES = 100_000
L2_FLUSH_BYTES = 512 << 20


# ------------------------------------------------------------------ helpers

def _env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return json.load(f), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "sm_max_mhz": 1965.0}, "fallback"


class ClockSampler:
    """NVML sampler of SM clock + throttle reasons during the timed region."""

    REASONS = {
        "gpu_idle": 0x1, "applications_clocks_setting": 0x2, "sw_power_cap": 0x4, "hw_slowdown": 0x8,
        "sync_boost": 0x10, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
        "hw_power_brake_slowdown": 0x80, "display_clock_setting": 0x100,
    }

    def __init__(self, index: int, period: float = 0.05):
        self.index, self.period = index, period
        self.samples, self.reasons = [], set()
        self._stop = threading.Event()
        self._thr = None
        self.max_mhz = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self._nv = None

    def _run(self):
        nv = self._nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
                mask = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                for k, v in self.REASONS.items():
                    if mask & v and k != "gpu_idle":
                        self.reasons.add(k)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self._nv is not None:
            self._thr = threading.Thread(target=self._run, daemon=True)
            self._thr.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._thr is not None:
            self._thr.join()

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": len(self.samples)}


def _flops_per_tile_eval(dims, m, r, AT, G, BT):
    """Algorithmic work of one tile evaluation with the template's structural zeros skipped
    (SURVEY §8(d)): FMAs of the canonical O5 chains whose coefficient is non-zero, plus the
    Hadamard multiplies; FLOP = 2 FMA + MUL.  Also returns the dense FMA count."""
    n = m + r - 1
    nz = lambda M: int(np.count_nonzero(M))
    if dims == 1:
        fma = nz(G) + nz(BT) + nz(AT)
        dense = n * r + n * n + m * n
        mul = n
    else:
        fma = (r + n) * nz(G) + 2 * n * nz(BT) + (n + m) * nz(AT)
        dense = n * r * r + n * n * r + 2 * n * n * n + m * n * n + m * m * n
        mul = n * n
    return 2 * fma + mul, fma, dense, mul


def _huffman_ops_per_tile_eval(m, r, AT, G, BT):
    """Huffman-order 2D tile evaluation (reading R21): one FMUL per non-zero coefficient use
    (the FMA count of _flops_per_tile_eval) and per Hadamard element, one FADD per tree node
    = uses minus the non-empty dot products.  Every op is one FP32-pipe lane-op."""
    n = m + r - 1
    rows = lambda M: int(np.count_nonzero(np.any(M != 0, axis=1)))
    _, fma, _, mul = _flops_per_tile_eval(2, m, r, AT, G, BT)
    dots = (r + n) * rows(G) + 2 * n * rows(BT) + (n + m) * rows(AT)
    return fma + mul + (fma - dots)


# ------------------------------------------------------------------ reference arm / cpu baseline

def oracle_sample_run(specs, every: int):
    """Time the oracle (as it stands) on every `every`-th candidate of each sweep, all tiles.
    Returns (tile_evals, seconds, threads, sample description)."""
    from oracle import points as OP, ref
    ref.lib()
    threads = ref.max_threads()
    evals = 0
    dt = 0.0
    for sp in specs:
        d, g = synth.random_tiles(sp.n_tiles, sp.dims, sp.n, sp.r, sp.dist, sp.seed)
        t0 = time.perf_counter()
        sets = [OP.f43_c(float(c)) for c in sp.params[::every]]
        ref.sweep(sp.dims, sp.m, sp.r, sets, d, g)
        dt += time.perf_counter() - t0
        evals += len(sets) * sp.n_tiles
    desc = (f"every {every}th of {N_C} c (={len(specs[0].params[::every])} c) x {specs[0].n_tiles} tiles x "
            f"{len(specs)} sweeps, oracle/ref.c OpenMP")
    return evals, dt, threads, desc


def run_reference(args, rank, world):
    """--impl reference: the oracle on the host cores is the reference arm (tier framing)."""
    if rank != 0:
        return 0
    from paper_2201_10369_b200.sweep import cfg2_specs
    specs = cfg2_specs(synth.c_grid(N_C), args.n_tiles)
    every = args.ref_every
    for _ in range(max(0, args.warmup)):
        oracle_sample_run(specs, every * 8)
    times, evals, threads, desc = [], 0, 1, ""
    for _ in range(args.steps):
        evals, dt, threads, desc = oracle_sample_run(specs, every)
        times.append(dt)
    tot = sum(times)
    value = evals * len(times) / tot
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "tile-evals/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / len(times),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic",
        "config": {"workload": "configs[1] c-sweep (bounded sample per step)", "n_c": N_C, "n_tiles": args.n_tiles,
                   "sweeps": [s.name for s in specs], "template": "{0,±c,±1/c,inf} F(4,3)"},
        "cpu_baseline": {"value": value, "unit": "tile-evals/s", "cores": threads, "kind": "oracle", "sample": desc},
        "e2e": {"value": value, "unit": "tile-evals/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ native arm

def bench_layer(torch, dev, flush, steps=10, rank=0, world=1, dist=None):
    """configs[2]: F(6x6,3x3) layer, N=32 C=K=256 56x56 pad 1, X16 points; unscored + scored.
    With world > 1 the batch is sharded over the ranks: rank r runs images
    [lo, hi); every timed iteration starts after a barrier and its time is the max over
    ranks; scored statistics are all-reduced (SUM of sums, MAX of maxs)."""
    from paper_2201_10369_b200 import api, points as PP
    from paper_2201_10369_b200.sweep import shard
    N, C, H, W, K, r, pad, m = 32, 256, 56, 56, 256, 3, 1, 6
    x, w = synth.layer_inputs(N, C, H, W, K, r, "normal", "he", seed=0)
    lo, hi = shard(N, rank, world)
    Nr = hi - lo
    xd, wd = torch.from_numpy(x[lo:hi]).to(dev), torch.from_numpy(w).to(dev)
    pts = PP.family_n8_cd(2.0, 1.003)
    Ho, Wo = H, W
    y = torch.empty((Nr, K, Ho, Wo), dtype=torch.float32, device=dev)
    ws = torch.empty(api.wino_conv2d_workspace_bytes(Nr, C, H, W, K, r, pad, m), dtype=torch.uint8, device=dev)

    def sync_ranks():
        if dist is not None:
            dist.barrier(device_ids=[dev.index])

    def max_over_ranks(vals):
        if dist is None:
            return vals
        t = torch.tensor(vals, dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.cpu().tolist()
    sums = torch.zeros(5, dtype=torch.float64, device=dev)
    maxs = torch.zeros(2, dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream()
    for _ in range(3):
        api.wino_conv2d_fp32(xd, wd, y, pad, m, pts, ws)
    torch.cuda.synchronize()
    fams = ["layer_filter", "layer_input", "layer_gemm", "layer_output"]
    # the layer time is measured with the library's per-launch event hook OFF (its events
    # serialise the layer's programmatic-dependent-launch chain); the per-kernel breakdown
    # comes from a second pass with the hook on
    ts = []
    for hook in (False, True):
        api.wino_timing_reset()
        api.wino_timing_enable(hook)
        for _ in range(steps):
            flush()
            sync_ranks()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            api.wino_conv2d_fp32(xd, wd, y, pad, m, pts, ws)
            b.record(stream)
            b.synchronize()
            if not hook:
                ts.append(a.elapsed_time(b))
    kern = {f: api.wino_timing_read(f)[0] / steps for f in fams}
    api.wino_timing_reset()
    api.wino_timing_enable(False)
    # scored (fp64 direct scoring on every output)
    sc = []
    for _ in range(2):
        flush()
        sync_ranks()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        api.wino_conv2d_fp32(xd, wd, y, pad, m, pts, ws, sums, maxs)
        b.record(stream)
        b.synchronize()
        sc.append(a.elapsed_time(b))
    api.wino_timing_enable(True)
    # NEXT row N3: the tcgen05 kind::tf32 contraction variants (not the parity path)
    def run_variant(flag, gemm_family):
        tv = []
        api.wino_timing_reset()
        for _ in range(steps):
            flush()
            sync_ranks()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            api.wino_conv2d_fp32(xd, wd, y, pad, m, pts, ws, flags=flag)
            b.record(stream)
            b.synchronize()
            tv.append(a.elapsed_time(b))
        kv = {f: api.wino_timing_read(f)[0] / steps
              for f in ["layer_filter", "layer_input", gemm_family, "layer_output"]}
        sv = torch.zeros(5, dtype=torch.float64, device=dev)
        mv = torch.zeros(2, dtype=torch.float64, device=dev)
        api.wino_conv2d_fp32(xd, wd, y, pad, m, pts, ws, sv, mv, flags=flag)
        torch.cuda.synchronize()
        if dist is not None:
            dist.all_reduce(sv, op=dist.ReduceOp.SUM)
        return max_over_ranks(tv), kv, sv.cpu().numpy()

    tf, kern_tf, s_tf = run_variant(api.WINO_CONV_TF32, "layer_gemm_tf32")
    tf3, kern_tf3, s_tf3 = run_variant(api.WINO_CONV_3XTF32, "layer_gemm_3xtf32")
    api.wino_timing_enable(False)
    ts, sc = max_over_ranks(ts), max_over_ranks(sc)
    if dist is not None:
        dist.all_reduce(sums, op=dist.ReduceOp.SUM)
        dist.all_reduce(maxs, op=dist.ReduceOp.MAX)
    s = sums.cpu().numpy() / 2
    t = statistics.median(ts)
    direct_flop = 2.0 * N * K * C * Ho * Wo * r * r
    # roofline: algorithmic FP32 work (GEMM MACs + zero-skipped transform FMAs) and fused bytes
    AT, G, BT = api.wino_points_to_matrices(m, r, pts)
    n = m + r - 1
    th = tw = (Ho + m - 1) // m
    T = N * th * tw
    gemm_mac = n * n * K * C * T
    nzG, nzB, nzA = (int(np.count_nonzero(M)) for M in (G, BT, AT))
    tr_fma = K * C * (r + n) * nzG + C * T * 2 * n * nzB + K * T * (n + m) * nzA
    f_alg = 2.0 * (gemm_mac + tr_fma)
    b_alg = 4.0 * (x.size + w.size + N * K * Ho * Wo)
    # tf32 GEMM kernel: algorithmic HBM bytes = read U and V once, write M once (padded sizes)
    Cp, Kp, Tp = -(-C // 32) * 32, -(-K // 128) * 128, -(-T // 256) * 256
    gemm_bytes = 4.0 * n * n * (Cp * Kp + Cp * Tp + Kp * Tp)
    g_ms = kern_tf["layer_gemm_tf32"]
    peaks, psrc = _peaks()
    t_tf = statistics.median(tf)
    tf32 = {
        "ms": t_tf, "effective_tflops": direct_flop / (t_tf * 1e-3) / 1e12, "kernel_ms": kern_tf,
        "gemm_tflops": 2.0 * gemm_mac / (g_ms * 1e-3) / 1e12 if g_ms else None,
        "gemm_roofline": {"bound": "hbm", "achieved_gbs": gemm_bytes / (g_ms * 1e-3) / 1e9 if g_ms else None,
                          "peak_gbs": peaks["hbm_gbs"], "peak_source": psrc,
                          "frac": gemm_bytes / (g_ms * 1e-3) / 1e9 / peaks["hbm_gbs"] if g_ms else None},
        "scored_mae": float(s_tf[0] / s_tf[3]) if s_tf[3] else None,
        "note": "WINO_CONV_TF32: tcgen05.mma kind::tf32 (TMA-fed, TMEM accumulators); operands rounded to "
                "TF32, so NOT the fp32 parity path -- reported separately",
    }
    t_tf3 = statistics.median(tf3)
    g3 = kern_tf3["layer_gemm_3xtf32"]
    gemm_bytes3 = 4.0 * n * n * (2 * Cp * Kp + 2 * Cp * Tp + Kp * Tp)   # hi + lo planes of U and V
    tf32x3 = {
        "ms": t_tf3, "effective_tflops": direct_flop / (t_tf3 * 1e-3) / 1e12, "kernel_ms": kern_tf3,
        "gemm_tflops": 2.0 * gemm_mac / (g3 * 1e-3) / 1e12 if g3 else None,
        "gemm_roofline": {"bound": "hbm", "achieved_gbs": gemm_bytes3 / (g3 * 1e-3) / 1e9 if g3 else None,
                          "peak_gbs": peaks["hbm_gbs"], "peak_source": psrc,
                          "frac": gemm_bytes3 / (g3 * 1e-3) / 1e9 / peaks["hbm_gbs"] if g3 else None},
        "scored_mae": float(s_tf3[0] / s_tf3[3]) if s_tf3[3] else None,
        "note": "WINO_CONV_3XTF32: hi/lo split, 3 tcgen05 MMAs per step; ~fp32 accuracy, not bitwise parity",
    }
    return {
        "workload": "configs[2] F(6x6,3x3) N=32 C=K=256 56x56 pad 1, points {0,±2,±1/2,-1/1.003,1.003,inf}",
        "parallelism": f"batch sharded over {world} ranks ({Nr} images on rank {rank}); time = max over ranks",
        "ms": t, "ms_min": min(ts), "effective_tflops": direct_flop / (t * 1e-3) / 1e12,
        "kernel_ms": kern, "flop_alg": f_alg, "bytes_alg": b_alg,
        "scored_ms": statistics.median(sc), "scored_mae": float(s[0] / s[3]) if s[3] else None,
        "l2": "flushed (512 MB write) before every run",
        "tf32_variant": tf32,
        "tf32x3_variant": tf32x3,
    }, f_alg, b_alg, t


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["native", "reference"], default="native")
    ap.add_argument("--n-tiles", type=int, default=N_TILES)
    ap.add_argument("--ref-every", type=int, default=32, help="--impl reference: every k-th candidate per step")
    ap.add_argument("--cpu-every", type=int, default=4,
                    help="cpu_baseline sample: every k-th candidate (~12 s of host work at 16 cores)")
    ap.add_argument("--no-layer", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 0)

    world = _env_int("WORLD_SIZE", 1)
    rank = _env_int("RANK", 0)
    local = _env_int("LOCAL_RANK", 0)

    if args.impl == "reference":
        return run_reference(args, rank, world)

    import torch
    import torch.distributed as dist
    from paper_2201_10369_b200 import api
    from paper_2201_10369_b200.sweep import cfg2_specs, make_rank_sweep, run_step

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    # WINO_FORCE_COLLECTIVES=1: initialise NCCL and run every collective of the N > 1 path
    # also with one rank (torchrun --nproc-per-node 1) -- a 1-GPU box exercises the NCCL code
    dist_on = world > 1 or os.environ.get("WINO_FORCE_COLLECTIVES") == "1"
    if dist_on:
        import datetime
        # finite timeout: a rank that dies makes the others fail instead of hanging the box
        dist.init_process_group("nccl", device_id=dev, timeout=datetime.timedelta(seconds=300))
    api.wino_supported(2, 4, 3)  # loads libwino.so (fails loudly if missing)

    specs = cfg2_specs(synth.c_grid(N_C), args.n_tiles)
    host = []
    rsw = []
    for sp in specs:
        d, g = synth.random_tiles(sp.n_tiles, sp.dims, sp.n, sp.r, sp.dist, sp.seed)
        host.append((d, g))
        rsw.append(make_rank_sweep(sp, rank, world, dev, d, g))
    stream = torch.cuda.current_stream()
    flush_buf = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device=dev)

    def flush():
        flush_buf.zero_()

    def barrier():
        if dist_on:
            dist.barrier(device_ids=[local])

    # ---- warm-up
    for _ in range(args.warmup):
        run_step(rsw)
    torch.cuda.synchronize()

    # ---- timed region (no timing hook: the library records no events here)
    step_ms = []
    launches = 0
    with ClockSampler(local) as clk:
        barrier()
        torch.cuda.synchronize()
        for _ in range(args.steps):
            flush()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            launches += run_step(rsw)
            b.record(stream)
            step_ms.append((a, b))
        torch.cuda.synchronize()
        barrier()
    step_ms = [a.elapsed_time(b) for a, b in step_ms]
    tot_ms = sum(step_ms)
    if dist_on:
        t = torch.tensor([tot_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        tot_ms = float(t.item())
    evals_per_step = sum(sp.n_cand * sp.n_tiles for sp in specs)
    value = evals_per_step * args.steps / (tot_ms * 1e-3)

    # ---- profiled pass: the same K steps again with the library's per-launch event hook on
    # (CUDA events recorded on each kernel's own launch stream) -> per-kernel times
    api.wino_timing_reset()
    api.wino_timing_enable(True)
    prof_ms = []
    barrier()
    torch.cuda.synchronize()
    for _ in range(args.steps):
        flush()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        run_step(rsw)
        b.record(stream)
        prof_ms.append((a, b))
    torch.cuda.synchronize()
    api.wino_timing_enable(False)
    prof_ms = [a.elapsed_time(b) for a, b in prof_ms]

    # dominant kernel (2D sweep) live timing -> roofline
    k2_ms, k2_n = api.wino_timing_read("sweep2d")
    k1_ms, _ = api.wino_timing_read("sweep1d")
    kref_ms, _ = api.wino_timing_read("sweep_refs2d")
    kfin_ms, _ = api.wino_timing_read("sweep_finalize")
    api.wino_timing_reset()
    sp2 = specs[2]
    AT, G, BT = api.wino_points_to_matrices(4, 3, sp2.point_sets(100, 101)[0])
    flop_te, fma_te, dense_te, mul_te = _flops_per_tile_eval(2, 4, 3, AT, G, BT)
    evals_2d = sum(rs.hi - rs.lo for rs in rsw if rs.spec.dims == 2) * sp2.n_tiles * args.steps
    peaks, peak_src = _peaks()
    nsm = torch.cuda.get_device_properties(dev).multi_processor_count
    fmax = float(peaks.get("sm_max_mhz", 1965.0))
    fp32_peak = nsm * 128 * 2 * fmax * 1e6 / 1e12
    achieved = evals_2d * flop_te / (k2_ms * 1e-3) / 1e12 if k2_ms > 0 else None
    traffic = None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        try:
            traffic = json.load(open(tp)).get("sweep2d_dram_bytes_per_launch")
        except Exception:
            traffic = None
    roofline = {
        "kernel": "sweep2d_reg_kernel<4,3> (K7, 2D F(4x4,3x3), tile pairs in registers)", "bound": "alu", "achieved": achieved,
        "peak": fp32_peak, "unit": "TFLOP/s", "frac": (achieved / fp32_peak) if achieved else None,
        "traffic": traffic,
        "peak_source": f"FP32 FFMA: {nsm} SMs x 128 lanes x 2 FLOP x {fmax:.0f} MHz (sm_max_mhz, {peak_src}); "
                       "microbench profiles/r01_pipes_microbench.jsonl measured 7.2e13",
        "flop_per_tile_eval": flop_te, "fma_per_tile_eval_zero_skipped": fma_te, "fma_per_tile_eval_dense": dense_te,
        "mul_per_tile_eval": mul_te, "kernel_ms_total": k2_ms, "launches": k2_n,
        "avg_launch_ms": k2_ms / k2_n if k2_n else None,
        "share_of_step": k2_ms / sum(prof_ms) if prof_ms else None,
        "timing": "CUDA events on the launch stream around each sweep call's PDL chain of candidate-chunk "
                  "launches of this kernel (events between chained launches would serialise them; 'launches' "
                  "counts the chained launches), in a second pass of the same K steps (the headline timed "
                  "region runs without the hook)",
        "profiled_pass_ms_per_step": statistics.mean(prof_ms) if prof_ms else None,
        "other_kernels_ms": {"sweep1d": k1_ms, "sweep_refs2d": kref_ms, "sweep_finalize": kfin_ms},
    }

    # ---- e2e: same job through the C-ABI with host tiles, H2D + D2H inside the timed region
    pinned = [(torch.from_numpy(d).pin_memory(), torch.from_numpy(g).pin_memory()) for d, g in host]
    out_host = [(torch.empty(rs.sums.shape, dtype=torch.float64).pin_memory(),
                 torch.empty(rs.maxs.shape, dtype=torch.float64).pin_memory()) for rs in rsw]
    h2d = sum(p[0].numel() * 4 + p[1].numel() * 4 for p in pinned)
    d2h = sum(o[0].numel() * 8 + o[1].numel() * 8 for o in out_host)
    e2e_ms, e2e_copy_ms, host_ms = [], [], []
    # The copies run on a side stream, one event per sweep: sweep k waits only for its own
    # tiles, so sweep k + 1's H2D overlaps sweep k's kernels (every copy is still inside the
    # timed region, which ends after the D2H of the statistics).  Both streams are created
    # streams: work on the legacy default stream would serialise with every copy.
    from paper_2201_10369_b200.sweep import abi_compute
    copy_stream = torch.cuda.Stream(device=dev)
    comp = torch.cuda.Stream(device=dev)
    barrier()
    torch.cuda.synchronize()
    for _ in range(args.steps):
        with torch.cuda.stream(comp):
            flush()
            a, c, b = (torch.cuda.Event(enable_timing=True) for _ in range(3))
            ready = {}
            a.record(comp)
            copy_stream.wait_stream(comp)
            with torch.cuda.stream(copy_stream):
                for rs, (pd, pg) in zip(rsw, pinned):
                    rs.d_tiles.copy_(pd, non_blocking=True)
                    rs.g_tiles.copy_(pg, non_blocking=True)
                    ready[id(rs)] = torch.cuda.Event()
                    ready[id(rs)].record(copy_stream)
                c.record(copy_stream)

            def compute_after_copy(rs):
                comp.wait_event(ready[id(rs)])
                abi_compute(rs)   # on the current stream = comp

            h0 = time.perf_counter()
            run_step(rsw, compute=compute_after_copy)
            host_ms.append(1e3 * (time.perf_counter() - h0))
            comp.wait_event(c)   # (already implied by the last sweep's wait; keeps the region closed)
            for rs, (hs, hm) in zip(rsw, out_host):
                hs.copy_(rs.sums, non_blocking=True)
                hm.copy_(rs.maxs, non_blocking=True)
            b.record(comp)
        b.synchronize()
        e2e_ms.append(a.elapsed_time(b))
        e2e_copy_ms.append(a.elapsed_time(c))
    torch.cuda.synchronize()
    e2e_tot = sum(e2e_ms)
    if dist_on:
        t = torch.tensor([e2e_tot], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_tot = float(t.item())
    e2e_value = evals_per_step * args.steps / (e2e_tot * 1e-3)

    # results of the job (rank 0 holds the reduced curve)
    from paper_2201_10369_b200.sweep import argmin_c, curve
    results = {}
    for rs in rsw:
        mae = curve(out_host[rsw.index(rs)][0].numpy())
        i, best = argmin_c(rs.spec.params, mae)
        results[rs.spec.name] = {"argmin_c": float(rs.spec.params[i]) if i is not None else None,
                                 "min_mae": best, "n_nonfinite_candidates": int(np.sum(~np.isfinite(mae)))}

    layer = None
    if not args.no_layer:
        layer, f_alg, b_alg, t_layer = bench_layer(torch, dev, flush, rank=rank, world=world,
                                                   dist=dist if dist_on else None)
        t_roof = max(f_alg / (fp32_peak * 1e12), b_alg / (float(peaks.get("hbm_gbs", 6458.7)) * 1e9)) / world
        layer["roofline_frac"] = t_roof / (t_layer * 1e-3)
        layer["roofline_bound"] = "fp32 FFMA (t_roof = max(F_alg/P_fp32, B_alg/BW_hbm))"

    # NEXT row N2: the Huffman-order and mixed-precision variants of the configs[1] 2D sweep, timed once
    variants = None
    if rank == 0 and world == 1 and not args.no_layer:
        variants = {}
        from paper_2201_10369_b200 import api
        sp = next(r for r in rsw if r.spec.dims == 2)
        sets, dd, gg = sp.sets, sp.d_tiles, sp.g_tiles           # the rank's shard = the whole job at N=1
        S, T = len(sets), sp.spec.n_tiles
        hws = torch.empty(api.wino_error_sweep_workspace_bytes(2, 4, 3, S, T), dtype=torch.uint8, device=dev)
        hs = torch.zeros((S, 5), dtype=torch.float64, device=dev)
        hm = torch.zeros((S, 2), dtype=torch.float64, device=dev)
        for vname, vflag, note in (("huffman_2d", api.WINO_SWEEP_HUFFMAN, "WINO_SWEEP_HUFFMAN (reading R21)"),
                                   ("mixed_2d", api.WINO_SWEEP_MIXED, "WINO_SWEEP_MIXED (reading R22)")):
            hs.zero_()
            hm.zero_()
            api.wino_error_sweep(2, 4, 3, sets, dd, gg, hs, hm, hws, flags=vflag)   # warm-up
            runs = []
            for _ in range(3):
                hs.zero_()
                hm.zero_()
                flush()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                api.wino_error_sweep(2, 4, 3, sets, dd, gg, hs, hm, hws, flags=vflag)
                b.record(stream)
                b.synchronize()
                runs.append(a.elapsed_time(b))
            hms = statistics.median(runs)
            mae = curve(hs.cpu().numpy())
            i, best = argmin_c(sp.spec.params, mae)
            variants[vname] = {
                "workload": f"configs[1] 2D {sp.spec.dist} sweep ({S} c x {T} tiles), {note}",
                "ms": hms, "ms_runs": runs, "value": S * T / (hms * 1e-3), "unit": "tile-evals/s",
                "argmin_c": float(sp.spec.params[i]) if i is not None else None, "min_mae": best}
            if vname == "huffman_2d":
                ops = _huffman_ops_per_tile_eval(4, 3, AT, G, BT)
                nsm_ = torch.cuda.get_device_properties(dev).multi_processor_count
                alu_peak = nsm_ * 128 * float(peaks.get("sm_max_mhz", 1965.0)) * 1e6 / 1e12
                ach = S * T * ops / (hms * 1e-3) / 1e12
                variants[vname]["kernel"] = ("run-time specialised register kernels, one per Huffman program class "
                                             "(NVRTC, huff_jit.cu); auto mode")
                variants[vname]["roofline"] = {
                    "bound": "alu", "achieved": ach, "peak": alu_peak, "unit": "Top/s", "frac": ach / alu_peak,
                    "fp32_ops_per_tile_eval": ops,
                    "peak_source": f"{nsm_} SMs x 128 FP32 lanes x 1 op (unfused FMUL / FADD) x sm_max_mhz"}
            if vname == "mixed_2d":
                # dense fp64 transforms: 2D F(4x4,3x3) = 6*3*3 + 6*6*3 + 6*6*6*2 + 4*6*6 + 4*4*6 DFMA
                dfma = 6 * 3 * 3 + 6 * 6 * 3 + 2 * 6 * 6 * 6 + 4 * 6 * 6 + 4 * 4 * 6
                nsm_ = torch.cuda.get_device_properties(dev).multi_processor_count
                fp64_peak = nsm_ * 64 * 2 * float(peaks.get("sm_max_mhz", 1965.0)) * 1e6 / 1e12
                ach = S * T * dfma * 2 / (hms * 1e-3) / 1e12
                variants[vname]["roofline"] = {
                    "bound": "fp64", "achieved": ach, "peak": fp64_peak, "unit": "TFLOP/s", "frac": ach / fp64_peak,
                    "dfma_per_tile_eval": dfma,
                    "peak_source": f"{nsm_} SMs x 64 DFMA/clk x 2 FLOP x sm_max_mhz (microbench: DFMA at half the "
                                   "FFMA rate, profiles/r01_pipes_microbench.jsonl)"}
        del hws

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        evals_c, dt_c, thr, desc = oracle_sample_run(specs, args.cpu_every)
        cpu = {"value": evals_c / dt_c, "unit": "tile-evals/s", "cores": thr, "kind": "oracle", "sample": desc,
               "seconds": dt_c}

    if dist_on:
        dist.barrier(device_ids=[local])
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "tile-evals/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": tot_ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": "configs[1]: c-sweep F(4,3) 1D + F(4x4,3x3) 2D, {0,±c,±1/c,inf}, "
                                   f"{N_C} log-spaced c in [0.05,20], {args.n_tiles} tiles/sweep, "
                                   "uniform[-1,1] + N(0,1), scored vs fp64 direct",
                       "tile_evals_per_step": evals_per_step, "parallelism": f"candidates/{world} ranks",
                       "l2": "flushed (512 MB write) between timed steps; step inputs 46 MB < L2"},
            "roofline": roofline,
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": "tile-evals/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "ms_per_step": e2e_tot / args.steps,
                    "h2d_ms_per_step": statistics.mean(e2e_copy_ms),
                    "host_enqueue_ms_per_step": statistics.mean(host_ms)},
            "gpu_launches": launches,
            "clocks": clk.summary(),
            "step_ms": step_ms,
            "results": results,
            "layer": layer,
            "variants": variants,
        }
        print(json.dumps(line), flush=True)
    if dist_on:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
