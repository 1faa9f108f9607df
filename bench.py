#!/usr/bin/env python
"""bench.py — E-A-HALS outer iterations/s on the BASELINE.json headline config.

Workload (BASELINE.json configs[4], "C5"): dense synthetic m = n = 32768,
r = 128, X = W0·H0 + |N(0, 0.01²)| with W0, H0 ~ U[0,1) (the tiled generator,
csrc/io.cpp enmf_gen_tiled, seed 1), initial factors random_init(seed 2),
E-A-HALS hp = 3 (beta0 .5, eta 1.5, gamma 1.01, gamma_bar 1.005), FP64.  One step
= one outer iteration (engine.hpp:309-440).  The timed window is iterations
1..K of that trajectory in every arm (the warm-up runs W iterations of the same
problem beforehand and is discarded), so our arm, our end-to-end call and the
reference arm do exactly the same work — the same iterations with the same
inner sweep counts (tests/test_gpu_long.py pins the trajectory to the
reference).

Our arm prints one JSON line with value (device-timed it/s, HBM-resident X), e2e
(the C-ABI enmf_gpu_run_dense call on pinned host buffers, copies included),
roofline (the dominant kernel, timed with CUDA events on the engine's stream),
cpu_baseline (the reference path on a bounded sample on the host cores), clocks
and gpu_launches.

--impl reference: the reference's own CPU implementation of the path on all host
cores — the bit-exact multi-threaded replica of enmf::run/step (oracle/replica.c,
pinned bitwise to the unmodified reference, tests/test_oracle.py and
tests/golden/golden_long.json "c5check") — on the same data, timing the same
window of iterations 1..K.

Multi-GPU (torchrun, N > 1): ONE C5 problem sharded over the ranks (SURVEY
§8(e), paper_1805_06604_b200/dist.py): rank p holds X[:, J_p] and X[I_p, :] and
the factor shards; the engine exchanges factor shards, r×r partials and one
scalar per HALS sweep through CUDA-IPC peer memory (csrc/dist.cuh).  Strong
scaling: value = K / (max over ranks of the device time of K iterations).
The tiled generator builds exactly each rank's blocks of the same matrix.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

M = N = 32768
R = 128
METRIC = "E-A-HALS outer iters/sec + % roofline, 32768² r=128, 1/2/4/8 B200"
UNIT = "outer_iters/s"
FP64_PEAK_TFLOPS = 37.1      # measured DMMA m8n8k4 peak on this pool's B200 (profiles/r01_fp64_peak.txt)
FP64_PEAK_SRC = "measured FP64 DMMA.8x8x4 peak, profiles/r01_fp64_peak.txt (MEASURED_PEAKS.json has no FP64 entry)"
# DRAM bytes per HALS sweep inside sweep_tm: ncu --set full of one 16-sweep launch at C5 size,
# dram__bytes_read.sum + dram__bytes_write.sum = 79.85 + 395.90 MB (profiles/r02_sweep_tm_lookahead_ncu.txt):
# mostly the rows written back each sweep (H ping-pongs between two buffers for the speculative
# stall decision), C and H reads stay L2-resident
SWEEP_DRAM_BYTES = (79.853056e6 + 395.901952e6) / 16
# tcgen05 kind::i8 floor: 8192 MAC/cycle/SM (M=128 N≥128 MMAs at 100% in profiles/r02_umma_rate.txt)
INT8_PEAK_TOPS = 2 * 8192 * 148 * 1.965e9 / 1e12
INT8_PEAK_SRC = ("tcgen05 kind::i8 MMA floor measured on this pool's B200 (M=128, N>=128: 8192 MAC/cycle/SM, "
                 "profiles/r02_umma_rate.txt) at the 1965 MHz max SM clock; nominal dense 4500")
SEED_DATA, SEED_INIT = 1, 2


def cfg_c5(iters):
    import paper_1805_06604_b200 as E
    c = E.algorithm_config("e-ahals-hp3")
    c.max_outer_iterations = iters
    return c


def config_block(args, world):
    return {"workload": "C5: dense m=n=32768 r=128, X=W0·H0+|N(0,0.01²)|, E-A-HALS hp3 (BASELINE.json configs[4])",
            "m": M, "n": N, "r": R, "algorithm": "e-ahals-hp3", "precision": "fp64",
            "beta0": 0.5, "eta": 1.5, "gamma": 1.01, "gamma_bar": 1.005,
            "l2": "inputs larger than L2 (X = 8.59 GB FP64 vs 126 MB L2); no flush needed",
            "parallelism": f"sharded x{world} (X column+row blocks, peer-memory exchanges)" if world > 1
            else "single GPU"}


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md recipe)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.f = tempfile.NamedTemporaryFile(mode="w+", suffix=".csv", delete=False)
        self.p = None

    def start(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "200"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return None
        time.sleep(0.25)
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except Exception:
            self.p.kill()
        self.f.flush()
        rows = []
        with open(self.f.name) as fh:
            for line in fh:
                parts = [p.strip() for p in line.split(",")]
                if len(parts) >= 9:
                    rows.append(parts)
        os.unlink(self.f.name)
        if not rows:
            return None
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


# ------------------------------------------------------------ CPU baseline
def host_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def replica_window(threads, nskip, nsteps, world=1):
    """The reference path (the bit-exact multi-threaded replica of enmf::run/step,
    oracle/replica.c) on C5 itself: the seeded data, `nskip` untimed iterations, then `nsteps`
    timed ones; returns it/s of the timed window and its inner sweep counts."""
    import ctypes as C
    import numpy as np
    from oracle.oracle import Config, Iter, Oracle, preset
    orc = Oracle("port")
    fn = orc.lib.orc_time_window
    dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
    fn.argtypes = [dp, C.c_size_t, C.c_size_t, dp, dp, C.c_size_t, C.POINTER(Config), C.c_size_t, C.c_size_t,
                   C.POINTER(C.c_double), C.POINTER(Iter)]
    fn.restype = C.c_int
    x = orc.gen_tiled(M, N, R, SEED_DATA, threads=threads)
    w0, h0 = orc.random_init(M, N, R, SEED_INIT)
    cfg = preset("e-ahals-hp3", max_outer_iterations=nskip + nsteps)
    recs = (Iter * max(nsteps, 1))()
    sec = C.c_double()
    orc.threads = threads
    try:
        rc = fn(x, M, N, w0, h0, R, C.byref(cfg), nskip, nsteps, C.byref(sec), recs)
    finally:
        orc.threads = 1
    if rc:
        raise RuntimeError(f"replica run failed: {rc}")
    return {"value": nsteps / sec.value, "unit": UNIT, "cores": threads, "kind": "port",
            "seconds": sec.value,
            "sweeps_h": [recs[i].inner_h_count for i in range(nsteps)],
            "sweeps_w": [recs[i].inner_w_count for i in range(nsteps)],
            "last_relative_error": recs[nsteps - 1].relative_error if nsteps else None}


REPLICA_NOTE = ("the bit-exact multi-threaded replica of the reference's enmf::run/step (oracle/replica.c: every "
                "output element in the reference's summation order, OpenMP over independent elements; pinned bitwise "
                "to the unmodified reference compiled from /root/reference — tests/test_oracle.py, and on C5 "
                "iteration 1 in tests/golden/golden_long.json) — the reference itself is single-threaded "
                "(SPEC.md:303) at ~370 s per C5 iteration")


# --------------------------------------------------------------- reference arm
def run_reference(args, rank, world):
    if rank != 0:
        return 0
    threads = host_threads()
    res = replica_window(threads, 0, args.steps)
    value = res["value"]
    line = {"metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": res["seconds"] / args.steps * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (the seeded tiled C5 generator, the same matrix as our arm)",
            "config": dict(config_block(args, world), window=f"outer iterations 1..{args.steps} of the seeded C5 run",
                           host_threads=threads),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                             "sample": f"C5 itself, outer iterations 1..{args.steps} (the window our arm times), "
                                       f"on {threads} host threads: " + REPLICA_NOTE},
            "sweeps": {"h": res["sweeps_h"], "w": res["sweeps_w"]},
            "last_relative_error": res["last_relative_error"],
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------- our arm
def gen_data(rank, world):
    """This rank's X block(s) (product generator, csrc/io.cpp enmf_gen_tiled — the oracle's
    streams bit for bit) and initial factor shards, as host arrays."""
    from paper_1805_06604_b200 import data as Dt
    from paper_1805_06604_b200 import dist as D
    wi, hi = Dt.random_init(M, N, R, SEED_INIT)
    if world == 1:
        return (Dt.gen_tiled(M, N, R, SEED_DATA),), wi, hi
    r0, mp, c0, np_ = D.shard_bounds_py(M, N, rank, world)
    xs = (Dt.gen_tiled(M, N, R, SEED_DATA, cols=slice(c0, c0 + np_)),
          Dt.gen_tiled(M, N, R, SEED_DATA, rows=slice(r0, r0 + mp)))
    return xs, wi[r0:r0 + mp].copy(), hi[:, c0:c0 + np_].copy()


def direct_rel_error(x, w, h, rows=2048):
    """||X - W·H||_F / ||X||_F in FP64 on the device, in row blocks."""
    num = 0.0
    for i in range(0, x.shape[0], rows):
        d = x[i:i + rows] - w[i:i + rows] @ h
        num += float((d * d).sum())
    return (num / float((x * x).sum())) ** 0.5


def _make_context(E, dist_mod, local_rank, rank, world, xs, exchange):
    """Single-GPU Context with X loaded, or this rank's ShardedContext."""
    if world == 1:
        ctx = E.Context(local_rank)
        ctx.load_device(xs[0].data_ptr(), M, N)
        return ctx
    ctx = dist_mod.ShardedContext(local_rank, rank, world, M, N, R, exchange)
    ctx.load_sharded_device(xs[0].data_ptr(), xs[1].data_ptr())
    return ctx


def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist
    import paper_1805_06604_b200 as E
    from paper_1805_06604_b200 import dist as D

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    xh_np, wi_np, hi_np = gen_data(rank, world)
    xs = tuple(torch.from_numpy(x).to(dev) for x in xh_np)
    wi_s, hi_s = torch.from_numpy(wi_np).to(dev), torch.from_numpy(hi_np).to(dev)
    torch.cuda.synchronize()
    exchange = D.torch_exchange() if world > 1 else None
    ctx = _make_context(E, D, local_rank, rank, world, xs, exchange)
    # warm-up: W iterations of the same problem, discarded; the timed window is iterations 1..K
    # of a fresh begin (the window the reference arm and the end-to-end call time)
    ctx.begin_device(wi_s.data_ptr(), hi_s.data_ptr(), R, cfg_c5(args.warmup))
    ctx.step(args.warmup)
    ctx.sync()
    ctx.end()
    prof_steps = 2
    cfg = cfg_c5(args.steps + prof_steps)
    ctx.begin_device(wi_s.data_ptr(), hi_s.data_ptr(), R, cfg)
    ctx.sync()
    stream = torch.cuda.ExternalStream(ctx.stream, device=dev)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    launches0 = ctx.kernel_launches
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clk = ClockSampler(local_rank)
    clk.start()
    e0.record(stream)
    ctx.step(args.steps)
    e1.record(stream)
    e1.synchronize()
    torch.cuda.synchronize()
    clocks = clk.stop()
    ms = e0.elapsed_time(e1)
    recs = ctx.sync()
    launches = ctx.kernel_launches - launches0
    if world > 1:
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    timed = recs[1: 1 + args.steps]
    sweeps_h = [r.inner_h_count for r in timed]
    sweeps_w = [r.inner_w_count for r in timed]
    # dominant kernel: FP64 DMMA GEMM, timed per phase with CUDA events on the engine stream
    phases = [ctx.step_profiled() for _ in range(prof_steps)]
    try:
        levels = tuple(ctx.digit_levels)   # INT8-digit levels S per product (0 = FP64 DMMA GEMM)
    except Exception:
        levels = (0, 0)
    recs = ctx.sync()
    w64 = torch.empty(wi_s.shape, dtype=torch.float64, device=dev)
    h64 = torch.empty(hi_s.shape, dtype=torch.float64, device=dev)
    ctx.end(w64.data_ptr(), h64.data_ptr())
    # TF32 variant (BASELINE configs[4]): same data, init and iteration count, the two cross
    # products on TF32 tensor cores; reported next to the FP64 line, not as its value
    tf32 = None
    if world == 1 and not args.no_tf32:
        cfg_t = cfg_c5(args.warmup)
        cfg_t.precision = E.Precision.tf32
        ctx.begin_device(wi_s.data_ptr(), hi_s.data_ptr(), R, cfg_t)   # warm-up (discarded)
        ctx.step(args.warmup)
        ctx.sync()
        ctx.end()
        cfg_t = cfg_c5(args.steps + prof_steps)
        cfg_t.precision = E.Precision.tf32
        ctx.begin_device(wi_s.data_ptr(), hi_s.data_ptr(), R, cfg_t)
        ctx.sync()
        t0e, t1e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        t0e.record(stream)
        ctx.step(args.steps)
        t1e.record(stream)
        t1e.synchronize()
        ctx.step(prof_steps)
        rt = ctx.sync()
        w32 = torch.empty_like(w64)
        h32 = torch.empty_like(h64)
        ctx.end(w32.data_ptr(), h32.data_ptr())
        tms = t0e.elapsed_time(t1e)
        # final factors judged by the direct residual ||X - WH|| / ||X|| in FP64 (the TF32 run's
        # in-loop estimate carries the tensor cores' FP32 accumulation bias, profiles/r01_tf32_bias.txt)
        f64_final, t_final = direct_rel_error(xs[0], w64, h64), direct_rel_error(xs[0], w32, h32)
        tf32 = {"value": args.steps / (tms * 1e-3), "unit": UNIT, "ms_per_step": tms / args.steps,
                "dtype": "tf32: cross products and HALS block products on TF32 tensor cores (X, H tiles in FP32); Grams, error, decisions FP64",
                "iterations": len(rt) - 1, "final_relative_error": t_final,
                "in_loop_estimate": rt[-1].relative_error,
                "fp64_final_relative_error": f64_final, "abs_diff": abs(t_final - f64_final),
                "within_1e-4": abs(t_final - f64_final) <= 1e-4,
                "restarts": int(sum(r.restarted for r in rt)), "fp64_restarts": int(sum(r.restarted for r in recs))}
    if world > 1:
        ctx.finalize()
    ctx.close()
    # dominant kernel: the persistent HALS sweep kernel (one launch per inner solve), timed per
    # phase with CUDA events on the engine stream; algorithmic work 2·r²·N per sweep
    ph = phases[-1]
    nh, mw = (N // world, M // world)
    sweep_ms = ph["update_h"] + ph["update_w"]
    sweep_flops = 2.0 * R * R * (nh * ph["sweeps_h"] + mw * ph["sweeps_w"])
    achieved = sweep_flops / (sweep_ms * 1e-3) / 1e12
    cross_ms = statistics.mean([(p["cross_wx"] + p["cross_xht"]) / 2 for p in phases])
    digit_gemms = statistics.mean([lv * (lv + 1) / 2 for lv in levels])
    cross_flops = 2.0 * R * M * N / world
    iter_ms = ms / args.steps
    flops_alg = 4.0 * M * N * R + 2.0 * (M + N) * R * R
    t_roof_ms = flops_alg / world / (FP64_PEAK_TFLOPS * 1e12) * 1e3
    value = args.steps / (ms * 1e-3)

    # e2e: the public API on pinned host buffers (single GPU: the drop-in C-ABI call
    # enmf_gpu_run_dense; sharded: load_sharded/begin/step/sync/end of this rank's blocks)
    e2e = None
    if not args.no_e2e:
        pin = lambda a: torch.empty(a.shape, dtype=torch.float64, pin_memory=True).copy_(torch.from_numpy(a))
        xh = [pin(x) for x in xh_np]
        wh, hh = pin(wi_np), pin(hi_np)
        del xs, xh_np
        torch.cuda.empty_cache()
        cfg2 = cfg_c5(args.steps)
        if world == 1:
            ctx2 = E.Context(local_rank)
        else:
            ctx2 = D.ShardedContext(local_rank, rank, world, M, N, R, exchange)
        xn = [x.numpy() for x in xh]
        wn, hn = wh.numpy(), hh.numpy()
        wout, hout = torch.empty_like(wh).pin_memory(), torch.empty_like(hh).pin_memory()
        # three whole calls on one context (the first also allocates the device buffers); the
        # median is reported, every call listed: a single call is at the mercy of one slow
        # cudaMalloc or page-in on a fresh box
        walls = []
        for _ in range(3):
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            t0 = time.perf_counter()
            if world == 1:
                rec2 = ctx2.run(xn[0], wn, hn, cfg2, E.TimingMode.none)
                fre = rec2.final_relative_error()
            else:
                ctx2.load_sharded(xn[0], xn[1])
                ctx2.begin(wn, hn, cfg2)
                ctx2.step(args.steps)
                rr = ctx2.sync()
                ctx2.end(wout.data_ptr(), hout.data_ptr())
                fre = rr[-1].relative_error
            t1 = time.perf_counter()
            w1 = t1 - t0
            if world > 1:
                t = torch.tensor([w1], device=dev, dtype=torch.float64)
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                w1 = float(t.item())
            walls.append(w1)
        wall = statistics.median(walls)
        if world > 1:
            ctx2.finalize()
        ctx2.close()
        xb = sum(x.numel() for x in xh) * 8
        e2e = {"value": args.steps / wall, "unit": UNIT,
               "h2d_bytes_per_step": int(xb + (wh.numel() + hh.numel()) * 8),
               "d2h_bytes_per_step": int((wh.numel() + hh.numel()) * 8 + (args.steps + 1) * 56),
               "step": (f"one enmf_gpu_run_dense call: X/W0/H0 host->device, {args.steps} outer iterations, "
                        f"W/H/records device->host (median of 3 calls)" if world == 1 else
                        f"per rank: X column+row blocks and factor shards host->device, {args.steps} outer "
                        f"iterations, factor shards/records device->host"),
               "seconds": wall, "calls_s": walls, "final_relative_error": fre}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            th = min(host_threads(), args.cpu_threads)
            res = replica_window(th, 0, 1)
            cpu = {"value": res["value"], "unit": UNIT, "cores": th, "kind": "port",
                   "sample": ("C5 itself, outer iteration 1 only (bounded sample; its sweeps "
                              f"{res['sweeps_h'][0]}+{res['sweeps_w'][0]} are fewer than a later iteration's), on "
                              f"{th} host threads: " + REPLICA_NOTE + "; bench.py --impl reference times the full window"),
                   "seconds": res["seconds"]}
        except Exception as ex:  # reported, never fatal for the GPU number
            cpu = {"error": str(ex)}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": iter_ms, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (the seeded tiled C5 generator, csrc/io.cpp enmf_gen_tiled)",
                "config": dict(config_block(args, world),
                               window=f"outer iterations 1..{args.steps} of the seeded C5 run (after a discarded "
                                      f"{args.warmup}-iteration warm-up run)"),
                "roofline": {"bound": "tensor",
                             "kernel": "hals::sweep_tm (persistent FP64 DMMA HALS sweeps with the iterate held "
                                       "in tensor memory, one launch per inner solve; 2·r²·N flop per sweep)",
                             "achieved": achieved, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                             "frac": achieved / FP64_PEAK_TFLOPS, "traffic": (args.traffic if args.traffic is not None else SWEEP_DRAM_BYTES * (ph["sweeps_h"] + ph["sweeps_w"]) / 2),
                             "traffic_note": "DRAM bytes per launch (one inner solve), from the ncu --set full capture's "
                                             "bytes per sweep (profiles/r02_sweep_tm_lookahead_ncu.txt, 30 MB: the rows written "
                                             "back each sweep); the iterate lives in tensor memory and C is read from L2",
                             "peak_source": FP64_PEAK_SRC, "launch_ms": sweep_ms / 2,
                             "cross_products": {
                                 "kernel": "FP64-accurate W_yᵀX / X·Tᵀ on the hand-written tcgen05 kind::i8 "
                                           "CTA-pair kernel (ozk::gemm_pair): S 8-bit digits per operand, one "
                                           "cta_group::2 MMA forms two digit pairs (factor digits p, p+1 x one "
                                           "X digit split over the pair), level sums in TMEM, exact offset "
                                           "corrections, truncation-bias estimate, FP64 recombination",
                                 "digit_levels": list(levels), "digit_products": digit_gemms,
                                 "ms": cross_ms, "fp64_equiv_tflops": cross_flops / (cross_ms * 1e-3) / 1e12,
                                 "int8_tops": (digit_gemms * cross_flops / (cross_ms * 1e-3) / 1e12
                                               if digit_gemms else None),
                                 "int8_peak_tops": INT8_PEAK_TOPS, "int8_peak_source": INT8_PEAK_SRC},
                             "iteration": {"flops_alg": flops_alg, "t_roof_ms": t_roof_ms,
                                           "frac": t_roof_ms / iter_ms,
                                           "note": "t_roof = (4mnr + 2(m+n)r²)/P at the FP64 DMMA peak; HALS "
                                                   "sweeps excluded; the cross products run on INT8 tensor "
                                                   "cores, which is how frac can pass what FP64 DMMA allows"},
                             "phases_ms": phases[-1]},
                "e2e": e2e, "cpu_baseline": cpu, "clocks": clocks, "gpu_launches": launches,
                "tf32_variant": tf32,
                "sweeps": {"h_mean": statistics.mean(sweeps_h) if sweeps_h else None,
                           "w_mean": statistics.mean(sweeps_w) if sweeps_w else None},
                "final_relative_error": recs[-1].relative_error if recs else None}
        print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------ C4 (CSR) workload
def gen_docs_csr(m, n, seed):
    """BASELINE configs[3]: n documents over m terms, document lengths lognormal(5, 1), term ids
    Zipf(1.1) (truncated to m), tf-idf weights, each column (document) L2-normalised; CSR over
    terms (rows).  Seeded numpy; the same description as the oracle's generator, not its stream."""
    import numpy as np
    rng = np.random.default_rng(seed)
    lens = np.maximum(1, rng.lognormal(5.0, 1.0, n).astype(np.int64))
    ranks = np.arange(1, m + 1, dtype=np.float64)
    p = ranks ** -1.1
    p /= p.sum()
    rows, cols, tf = [], [], []
    for j in range(n):
        t = rng.choice(m, size=int(lens[j]), p=p)
        u, c = np.unique(t, return_counts=True)
        rows.append(u); cols.append(np.full(u.size, j)); tf.append(c.astype(np.float64))
    rows = np.concatenate(rows); cols = np.concatenate(cols); tf = np.concatenate(tf)
    df = np.bincount(rows, minlength=m).astype(np.float64)
    v = tf * np.log(n / np.maximum(df[rows], 1.0))
    v = np.where(v > 0, v, 1e-12)
    norm = np.sqrt(np.bincount(cols, weights=v * v, minlength=n))
    v = v / norm[cols]
    order = np.lexsort((cols, rows))
    rows, cols, v = rows[order], cols[order], v[order]
    off = np.zeros(m + 1, dtype=np.uint64)
    np.add.at(off, rows + 1, 1)
    return np.cumsum(off).astype(np.uint64), cols.astype(np.uint64), v


def run_c4(args):
    import numpy as np
    import torch
    import paper_1805_06604_b200 as E
    m, n, r = 30000, 10000, 20
    off, cidx, vals = gen_docs_csr(m, n, 404)
    rng = np.random.default_rng(405)
    w0, h0 = rng.random((m, r)), rng.random((r, n))
    cfg = E.algorithm_config("e-ahals-hp3")
    cfg.max_outer_iterations = args.warmup + args.steps
    ctx = E.Context(0)
    ctx.load_csr(off, cidx, vals, m, n)
    ctx.begin(w0, h0, cfg)
    ctx.step(args.warmup)
    ctx.sync()
    stream = torch.cuda.ExternalStream(ctx.stream, device=torch.device("cuda", 0))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    ctx.step(args.steps)
    e1.record(stream)
    e1.synchronize()
    ms = e0.elapsed_time(e1)
    recs = ctx.sync()
    ctx.end()
    cfg2 = E.algorithm_config("e-ahals-hp3")
    cfg2.max_outer_iterations = args.steps
    t0 = time.perf_counter()
    rec2 = ctx.run_csr(off, cidx, vals, m, n, w0, h0, cfg2, E.TimingMode.none)
    wall = time.perf_counter() - t0
    ctx.close()
    cpu = None
    if not args.no_cpu:
        from oracle.oracle import Oracle, preset
        orc = Oracle("reference")
        k = 3
        t0 = time.perf_counter()
        orc.run_csr(off, cidx, vals, m, n, w0, h0, preset("e-ahals-hp3", max_outer_iterations=k))
        t1 = time.perf_counter()
        orc.run_csr(off, cidx, vals, m, n, w0, h0, preset("e-ahals-hp3", max_outer_iterations=0))
        t2 = time.perf_counter()
        cpu = {"value": k / max((t1 - t0) - (t2 - t1), 1e-9), "unit": UNIT, "cores": 1, "kind": "reference",
               "sample": f"{k} outer iterations of enmf::run<SparseMatrix> on the same C4 matrix (setup time "
                         f"subtracted via a 0-iteration run); one run is single-threaded in the reference"}
    line = {"metric": "E-A-HALS outer iters/sec, C4 CSR 30000×10000 r=20", "value": args.steps / (ms * 1e-3),
            "unit": UNIT, "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic CSR (lognormal(5,1) document lengths, Zipf(1.1) terms, tf-idf, L2 columns)",
            "config": {"workload": "C4: BASELINE.json configs[3]", "m": m, "n": n, "r": r, "nnz": int(vals.size),
                       "algorithm": "e-ahals-hp3"},
            "e2e": {"value": args.steps / wall, "unit": UNIT, "seconds": wall,
                    "h2d_bytes_per_step": int(vals.size * 16 + (m + 1) * 8 + (m + n) * r * 8),
                    "d2h_bytes_per_step": int((m + n) * r * 8)},
            "cpu_baseline": cpu, "final_relative_error": recs[-1].relative_error,
            "sweeps": {"h_mean": statistics.mean(r_.inner_h_count for r_ in recs[1:]),
                       "w_mean": statistics.mean(r_.inner_w_count for r_ in recs[1:])}}
    print(json.dumps(line), flush=True)
    return 0


def gen_dense_config(which, seed):
    """BASELINE configs[1] (C2) / configs[2] (C3) as seeded numpy data (same descriptions as the
    oracle's generators, not their streams)."""
    import numpy as np
    rng = np.random.default_rng(seed)
    if which == "c2":   # image-shaped: 10304 pixels × 400 images, r = 40, 70%-sparse W0, |N(0,.01²)|, rescaled
        m, n, r = 10304, 400, 40
        w = rng.random((m, r)) * (rng.random((m, r)) >= 0.7)
        x = w @ rng.random((r, n)) + np.abs(0.01 * rng.standard_normal((m, n)))
        x /= x.max()
        return x, r, "e-ahals-hp3", 500
    m = n = 2000
    r = 30
    x = rng.random((m, r)) @ rng.random((r, n))
    x = np.maximum(x + 0.05 * x.mean() * rng.standard_normal((m, n)), 0.0)
    return x, r, "e-anls-hp1", 100


def run_dense_config(args):
    import numpy as np
    import torch
    import paper_1805_06604_b200 as E
    x, r, alg, iters = gen_dense_config(args.workload, 505)
    m, n = x.shape
    rng = np.random.default_rng(506)
    w0, h0 = rng.random((m, r)), rng.random((r, n))
    steps = min(args.steps, iters)
    cfg = E.algorithm_config(alg)
    cfg.max_outer_iterations = args.warmup + steps
    ctx = E.Context(0)
    ctx.load(x)
    ctx.begin(w0, h0, cfg)
    ctx.step(args.warmup)
    ctx.sync()
    stream = torch.cuda.ExternalStream(ctx.stream, device=torch.device("cuda", 0))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    ctx.step(steps)
    e1.record(stream)
    e1.synchronize()
    ms = e0.elapsed_time(e1)
    recs = ctx.sync()
    ctx.end()
    cfg2 = E.algorithm_config(alg)
    cfg2.max_outer_iterations = iters
    t0 = time.perf_counter()
    rec2 = ctx.run(x, w0, h0, cfg2, E.TimingMode.none)
    wall = time.perf_counter() - t0
    ctx.close()
    cpu = None
    if not args.no_cpu:
        from oracle.oracle import Oracle, preset
        orc = Oracle("reference")
        k = 5 if args.workload == "c2" else 2
        t0 = time.perf_counter()
        orc.run_dense(x, w0, h0, preset(alg, max_outer_iterations=k))
        t1 = time.perf_counter()
        orc.run_dense(x, w0, h0, preset(alg, max_outer_iterations=0))
        t2 = time.perf_counter()
        cpu = {"value": k / max((t1 - t0) - (t2 - t1), 1e-9), "unit": UNIT, "cores": 1, "kind": "reference",
               "sample": f"{k} outer iterations of enmf::run on the same matrix (setup subtracted via a "
                         f"0-iteration run); one run is single-threaded in the reference"}
    line = {"metric": f"{alg} outer iters/sec, {args.workload.upper()} {m}×{n} r={r}",
            "value": steps / (ms * 1e-3), "unit": UNIT, "n_gpus": 1, "steps": steps, "warmup": args.warmup,
            "ms_per_step": ms / steps, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (seeded numpy, BASELINE.json description)",
            "config": {"workload": f"{args.workload.upper()}: BASELINE.json configs[{1 if args.workload == 'c2' else 2}]",
                       "m": m, "n": n, "r": r, "algorithm": alg},
            "e2e": {"value": iters / wall, "unit": UNIT, "seconds": wall, "iterations": iters,
                    "h2d_bytes_per_step": int((m * n + (m + n) * r) * 8),
                    "d2h_bytes_per_step": int((m + n) * r * 8)},
            "cpu_baseline": cpu, "final_relative_error": rec2.final_relative_error()}
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-tf32", action="store_true")
    ap.add_argument("--workload", default="c5", choices=["c5", "c2", "c3", "c4"],
                    help="c5: the headline (default); c2 / c3 / c4: the other BASELINE configs (extra lines)")
    ap.add_argument("--cpu-threads", type=int, default=64)
    ap.add_argument("--traffic", type=float, default=None,
                    help="dram bytes per GEMM launch from an ncu --set full capture (profiles/)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, rank, world)
    if args.workload == "c4":
        return run_c4(args)
    if args.workload in ("c2", "c3"):
        return run_dense_config(args)
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    rc = run_ours(args, rank, world, local_rank)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    return rc


if __name__ == "__main__":
    sys.exit(main())
