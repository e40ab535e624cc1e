"""Benchmark of the B200-native Seven-League online path generator (BASELINE.json metric:
"7L path-steps/sec (device-timed) at 1/2/4/8 B200; % of tensor/FP32/HBM roofline").

Headline workload = BASELINE.json configs[4] (the scaling config, and the paper's own network shape,
PAPER.md:85): CIR kappa=1, Ybar=0.1, sigma=0.3, Y0=0.1, T=4, 32 steps of 0.125, m=7 Gauss-Hermite nodes,
[5,50,50,50,50,7] Softplus MLP with theta as network input (oracle-fitted weights), STATS output (fused
moments + 4096-bin histogram), tcgen05 bf16 MMAs (--prec).  One bench "step" = one sl7_simulate over the
rank's share of the paths:
  --scaling strong (default): 4e9 paths in total, rank r of N takes [r ceil(4e9/N), ...) (configs[4] as
                              written: at N=1 one GPU runs all 4e9 paths, 1.28e11 path-steps per step);
  --scaling weak:             5e8 paths per GPU (configs[4]'s per-GPU share at N=8).
Under torchrun the only collective is one NCCL all_reduce(SUM) of the fp64 statistics vector per step,
inside the timed region; the step time is the max over ranks.

At N=1 the line also carries "modes": the other BASELINE configs, each timed on the device the same way
(L2 flushed, CUDA events, NVML clocks) with its own algorithmic roofline:
  cfg3  exact-collocation GBM, FULL step-major [65][2e8] fp32 path tensor (52 GB): HBM-store-bound;
  cfg2  OU and CIR (the paper's process) in BF16 / TF32 / SPLIT / FP32, exact OU, CDC_PRED (OU also
        with fast normals) and the quantile-marginal 7L-CDC (OU);
  cfg4  the headline workload in TF32 / SPLIT / FP32 (1e8 paths; FP32 2.5e7) and with CDC_PRED;
  cfg1  the GBM dt sweep n = 1..64 (1e7 paths) in BF16 / TF32 / SPLIT / FP32 and exact GBM.

python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference] [--prec bf16|tf32|split|fp32]
                [--scaling strong|weak] [--paths P] [--no-modes] [--no-cpu-baseline]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "7L path-steps/sec (device-timed)"
UNIT = "path-steps/s"
N_BINS = 4096
L2_FLUSH_BYTES = 512 << 20   # > 126 MB L2
STRONG_TOTAL = 4_000_000_000
WEAK_PER_GPU = 500_000_000
CFG1_SWEEP = (1, 2, 4, 8, 16, 32, 64)
HIST = {"gbm": (0.0, 4.0), "ou": (-3.0, 3.0), "cir": (0.0, 0.8)}

# Algorithmic work per path-step: what the method must do, not what a kernel
# issues.  Transcendental activations = one per hidden unit (the XU roofline counts ONE MUFU op each, the
# least any implementation can spend); MLP FLOP with layer 1 folded to rank 1; RNG + interpolation
# instruction budgets for the issue-bound kernels: Philox4x32-10 / 4 normals = 11, Box-Muller 9 per normal,
# g_m product form 3(m-1) FMUL + 2m FFMA/FADD + 1 rcp, the CDC table interpolation in the state (basis
# 3(m-1) + 2m + 1, then m x m FFMA), the exact-GBM reference (1 FADD).
PHILOX_PER_NORMAL = 11
BOX_MULLER_PER_NORMAL = 9


def gm_instr(m):
    return 3 * (m - 1) + 2 * m + 1


def exact_instr(m):
    return PHILOX_PER_NORMAL + BOX_MULLER_PER_NORMAL + gm_instr(m) + 1


def exact_special_instr():
    # GBM closed-form g_m (Horner in X with shared coefficients, y_j = Y c_j): m FFMA + 1 FMUL; the store
    return PHILOX_PER_NORMAL + BOX_MULLER_PER_NORMAL + 6 + 1


def cdc_pred_instr(m):
    # the 7L-CDC step with predicted marginal points as ONE bivariate polynomial of degree m-1 in the clamped,
    # normalised state and in X (the same interpolant as the table-then-g_m form, R-26): m(m-1) + (m-1)
    # FMA, the clamp (2) and the state normalisation (1)
    return PHILOX_PER_NORMAL + BOX_MULLER_PER_NORMAL + m * (m - 1) + (m - 1) + 3


def cdc_pred_instr_lagrange(m):
    # the same step in the Lagrange forms of PAPER.md:106 / R-19: the basis in the state, the m x m contraction,
    # g_m at X
    return PHILOX_PER_NORMAL + BOX_MULLER_PER_NORMAL + gm_instr(m) + m * m + gm_instr(m) + 2


def ann_flops_per_path_step(dims):
    """Algorithmic FLOPs of one MLP evaluation with layer 1 folded to rank 1 (2 FLOP per MAC)."""
    f = 2 * dims[1]
    for l in range(1, len(dims) - 1):
        f += 2 * dims[l] * dims[l + 1]
    return f


# NVML throttle reasons that void a timed region (sw_power_cap is kept and only noted)
THROTTLE_REJECT = {"HwSlowdown", "HwThermalSlowdown", "SwThermalSlowdown", "HwPowerBrakeSlowdown"}


class ClockSampler(threading.Thread):
    """Samples SM clock and throttle reasons via NVML every 100 ms during the timed region."""

    def __init__(self, index):
        super().__init__(daemon=True)
        self.index = index
        self.samples, self.reasons = [], set()
        self.reason_counts = {}   # samples per reason (GpuIdle can appear in the gaps between timed launches)
        self.max_mhz = None
        self._halt = threading.Event()
        self.ok = True

    def run(self):
        try:
            import pynvml as N
            N.nvmlInit()
            h = N.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM)
            names = {getattr(N, k): k for k in dir(N) if k.startswith("nvmlClocksThrottleReason") and
                     isinstance(getattr(N, k), int)}
            while not self._halt.is_set():
                self.samples.append(N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM))
                r = N.nvmlDeviceGetCurrentClocksThrottleReasons(h)
                for bit, name in names.items():
                    if bit and bit != 0xFFFFFFFFFFFFFFFF and (r & bit) == bit and "All" not in name and "None" not in name:
                        nm = name.replace("nvmlClocksThrottleReason", "")
                        self.reasons.add(nm)
                        self.reason_counts[nm] = self.reason_counts.get(nm, 0) + 1
                time.sleep(0.1)
        except Exception as e:  # NVML missing: report, do not fake
            self.ok = False
            self.reasons.add("nvml_error:%s" % type(e).__name__)

    def stop(self):
        self._halt.set()
        self.join(timeout=2)

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "reason_samples": dict(sorted(self.reason_counts.items())),
                "samples": len(self.samples)}


def measured_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


# ------------------------------------------------------------------------------------------ oracle

def _oracle_chunk(args):
    import numpy as np
    from threadpoolctl import threadpool_limits
    threadpool_limits(1)                      # one BLAS thread per pool worker
    from oracle import sl7_oracle as O
    from sl7_inputs import load_golden_blob, workloads
    (wname, lo, n) = args
    w = workloads()[wname]
    net = O.parse_blob(load_golden_blob(w.blob))
    theta = tuple(w.theta) if w.process != "gbm" else ()
    paths = np.arange(lo, lo + n, dtype=np.uint64)
    spec = O.Spec(w.m, "ann", theta, w.y0, w.T / w.n_steps, w.n_steps, net=net)
    with np.errstate(all="ignore"):
        O.simulate(spec, w.seed, paths)
    return n * w.n_steps


def oracle_throughput(n_paths, wname="cfg4", reps=1):
    """Time the float64 oracle (as it stands) over a bounded path sample on all host cores; returns the
    path-steps/s of each repetition, the cores used and the elapsed seconds of each repetition."""
    import multiprocessing as mp
    cores = len(os.sched_getaffinity(0))
    chunk = max(1, -(-n_paths // cores))
    jobs = [(wname, lo, min(chunk, n_paths - lo)) for lo in range(0, n_paths, chunk)]
    for k in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ[k] = "1"
    ctx = mp.get_context("fork")
    rates, els = [], []
    with ctx.Pool(min(cores, len(jobs))) as pool:
        pool.map(_oracle_chunk, [(wname, 0, 64)] * min(cores, len(jobs)))   # warm the workers (imports)
        for _ in range(reps):
            t0 = time.perf_counter()
            done = sum(pool.map(_oracle_chunk, jobs))
            el = time.perf_counter() - t0
            rates.append(done / el)
            els.append(el)
    return rates, min(cores, len(jobs)), els


def headline_config(W, a, world, n_rank):
    return {"workload": "cfg4 (BASELINE configs[4]): CIR kappa=1 Ybar=0.1 sigma=0.3 Y0=0.1, T=4, 32 steps, m=7, "
                        "[5,50,50,50,50,7] softplus (theta as input), STATS (moments + 4096-bin histogram), "
                        "%s scaling: %s" % (a.scaling, "%.3g paths in total" % a.total if a.scaling == "strong"
                                              else "%.3g paths per GPU" % n_rank),
            "process": "cir", "theta": list(W.theta), "y0": W.y0, "T": W.T, "n_steps": W.n_steps, "m": W.m,
            "dims": list(W.dims), "paths_total": a.total if a.scaling == "strong" else n_rank * world,
            "paths_per_gpu": n_rank, "l2": "flushed (512 MiB write) before every timed step",
            "parallelism": "dp%d" % world}


# -------------------------------------------------------------------------------------------- main

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="sl7", choices=["sl7", "reference"])
    ap.add_argument("--prec", default="bf16", choices=["fp32", "bf16", "tf32", "split"])
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"])
    ap.add_argument("--paths", type=int, default=0,
                    help="strong: total paths (default 4e9); weak: paths per GPU (default 5e8)")
    ap.add_argument("--ref-paths", type=int, default=32768, help="oracle sample per reference-arm step")
    ap.add_argument("--no-modes", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    a = ap.parse_args()
    a.total = a.paths or STRONG_TOTAL

    from sl7_inputs import load_golden_blob, workloads
    W = workloads()["cfg4"]
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    from paper_2302_05170_b200.dist import max_over_ranks, strong_shard, weak_shard
    if a.scaling == "strong":
        offset, n_rank = strong_shard(a.total, rank, world)
    else:
        offset, n_rank = weak_shard(a.paths or WEAK_PER_GPU, rank)
    config = headline_config(W, a, world, n_rank)

    if a.impl == "reference":
        # the reference arm of this tier is the float64 oracle, timed on the host cores on a
        # bounded sample of the same workload; under torchrun rank 0 alone runs it
        if rank != 0:
            return
        rates, cores, els = oracle_throughput(a.ref_paths, "cfg4", reps=a.warmup + a.steps)
        t = els[a.warmup:]
        val = a.ref_paths * W.n_steps / statistics.mean(t)
        line = {"impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": a.gpus,
                "steps": a.steps, "warmup": a.warmup, "ms_per_step": 1e3 * statistics.mean(t),
                "higher_is_better": True, "scaling": a.scaling, "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (oracle-fitted weights)", "config": dict(config, paths_per_step=a.ref_paths),
                "cpu_baseline": {"value": val, "unit": UNIT, "cores": cores, "kind": "oracle",
                                 "sample": "%d paths x 32 steps of cfg4 per step (float64 numpy oracle, "
                                           "multiprocessing pool)" % a.ref_paths},
                "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    import torch
    import paper_2302_05170_b200 as sl7

    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl")
    sl7.load_library()
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream()
    ctx = sl7.Context(W.m, list(W.dims), W.act, device=local)
    ctx.load_weights(load_golden_blob(W.blob))
    P = {"fp32": sl7.PREC_FP32, "bf16": sl7.PREC_BF16, "tf32": sl7.PREC_TF32, "split": sl7.PREC_SPLIT}
    prec = P[a.prec]
    lo, hi = HIST["cir"]
    opts = sl7.make_opts(prec=prec, colloc=sl7.COLLOC_ANN, path_offset=offset, stream=stream, hist_lo=lo,
                         hist_hi=hi, shift=W.y0, n_bins=N_BINS)
    stats = torch.zeros(sl7.stats_elems(N_BINS), dtype=torch.float64, device=dev)
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device=dev)
    dt = W.T / W.n_steps

    def barrier():
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
            torch.cuda.synchronize()

    def step(ev=None):
        # one pass of the hot path over the rank's paths; the exchange step (one SUM all-reduce of the fp64
        # stats vector) is part of the step
        if ev is not None:
            ev[0].record(stream)
        ctx.simulate(W.y0, dt, W.n_steps, W.theta, n_rank, W.seed, sl7.OUT_STATS, opts, stats=stats)
        if ev is not None:
            ev[1].record(stream)
        if dist:
            dist.all_reduce(stats, op=dist.ReduceOp.SUM)
        if ev is not None:
            ev[2].record(stream)

    for _ in range(a.warmup):
        step()
    barrier()

    # ---------------- timed region: K steps, CUDA events on the launch stream; a region that saw a hardware /
    # thermal slowdown is measured once more (the contract's rule) and the line says so
    for attempt in range(2):
        clk = ClockSampler(local)
        clk.start()
        step_ms, kernel_ms = [], []
        barrier()
        for _ in range(a.steps):
            flush.fill_(1.0)                                     # L2 flush (untimed)
            ev = tuple(torch.cuda.Event(enable_timing=True) for _ in range(3))
            step(ev)
            torch.cuda.synchronize()
            kernel_ms.append(ev[0].elapsed_time(ev[1]))
            step_ms.append(ev[0].elapsed_time(ev[2]))
        barrier()
        clk.stop()
        throttled = bool(set(clk.reasons) & THROTTLE_REJECT)
        if dist:
            flag = torch.tensor([1.0 if throttled else 0.0], device=dev)
            dist.all_reduce(flag, op=dist.ReduceOp.MAX)
            throttled = flag.item() > 0
        if not throttled:
            break
    remeasured = attempt > 0
    t_step = max_over_ranks(statistics.mean(step_ms), dev)
    total_paths = a.total if a.scaling == "strong" else n_rank * world
    value = total_paths * W.n_steps / (t_step * 1e-3)
    summ = sl7.stats_summary(stats.cpu().numpy(), opts, q_levels=[0.01, 0.5, 0.99])

    # ---------------- e2e: the same step through the C ABI with HOST buffers (sl7_simulate_host_async: the
    # kernel parameters travel host->device with the launch, the stats vector comes back to pinned host
    # memory every step); sl7_sync ends each step
    h_st = torch.empty(sl7.stats_elems(N_BINS), dtype=torch.float64, pin_memory=True).numpy()
    e2e_ms, up_b, down_b = [], 0, 0
    for it in range(1 + a.steps):
        barrier()
        t0 = time.perf_counter()
        _, _, up_b, down_b = ctx.simulate_host_async(W.y0, dt, W.n_steps, W.theta, n_rank, W.seed, sl7.OUT_STATS,
                                                     opts, None, h_st)
        ctx.sync()
        if dist:
            hs = torch.from_numpy(h_st).to(dev)
            dist.all_reduce(hs, op=dist.ReduceOp.SUM)
            h_st[:] = hs.cpu().numpy()
            up_b += h_st.nbytes
            down_b += h_st.nbytes
        el = time.perf_counter() - t0
        if it:
            e2e_ms.append(el * 1e3)
    e2e_step = max_over_ranks(statistics.mean(e2e_ms), dev)

    if rank != 0:
        dist.destroy_process_group()
        return

    peaks = measured_peaks()
    sm_max = peaks.get("sm_max_mhz", 1965.0)
    n_sms = torch.cuda.get_device_properties(dev).multi_processor_count
    k_ms = statistics.mean(kernel_ms)
    rate_k = n_rank * W.n_steps / (k_ms * 1e-3)
    roof = ann_roofline(W.dims, prec, rate_k, sl7, peaks, n_sms, sm_max)
    # dram__bytes_read.sum + dram__bytes_write.sum of this kernel (ncu --set full, profiles/r02_cfg4_bf16_ncu.md):
    # in STATS mode nothing scales with the path count (weights + stats vector)
    roof["traffic"] = TRAFFIC.get(a.prec)
    roof["traffic_note"] = "dram bytes per launch from the ncu --set full capture (STATS mode: independent of N_P)"

    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps, "warmup": a.warmup,
            "ms_per_step": t_step, "higher_is_better": True, "scaling": a.scaling, "vs_baseline": None,
            "dtype": {"fp32": "f32", "bf16": "bf16", "tf32": "tf32", "split": "bf16x3"}[a.prec],
            "data": "synthetic (oracle-fitted weights)", "config": dict(config, prec=a.prec),
            "roofline": roof, "gpu_launches": 2 * a.steps,
            "gpu_launches_note": "per step: the stats zero-fill kernel + the fused 32-step ANN kernel",
            "clocks": dict(clk.summary(), remeasured=remeasured),
            "e2e": {"value": total_paths * W.n_steps / (e2e_step * 1e-3), "unit": UNIT, "h2d_bytes_per_step": up_b,
                    "d2h_bytes_per_step": down_b, "ms_per_step": e2e_step,
                    "api": "sl7_simulate_host_async + sl7_sync (pinned host stats buffer)"},
            "terminal": {"mean": summ["mean"], "var": summ["var"], "n": summ["n"], "n_nonfinite": summ["n_nonfinite"],
                         "quantiles_1_50_99": summ["quantiles"],
                         "cir_law": {"mean": 0.1, "var_T4": 0.0044985}},
            "kernel_ms_mean": k_ms}
    if world == 1 and not a.no_modes:
        del flush
        line["modes"] = run_modes(sl7, torch, dev, stream, peaks, n_sms, sm_max)
    if not a.no_cpu_baseline and world == 1:
        sample = 1048576
        rates, cores, els = oracle_throughput(sample, "cfg4", reps=1)
        line["cpu_baseline"] = {"value": rates[0], "unit": UNIT, "cores": cores, "kind": "oracle",
                                "sample": "%d paths x 32 steps of cfg4 (%.1f s), float64 numpy oracle, "
                                          "multiprocessing pool" % (sample, els[0])}
        # also a 1-core number (one chunk of the same oracle in this process, one BLAS thread)
        from threadpoolctl import threadpool_limits
        n1 = 65536
        with threadpool_limits(1):
            t0 = time.perf_counter()
            done = _oracle_chunk(("cfg4", 0, n1))
            el1 = time.perf_counter() - t0
        line["cpu_baseline"]["value_1core"] = done / el1
        line["cpu_baseline"]["sample_1core"] = "%d paths x 32 steps of cfg4 on one core (%.1f s)" % (n1, el1)
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


# ncu --set full DRAM bytes (read + write) per launch of the headline kernel, by precision
TRAFFIC = {"bf16": 129024}   # profiles/r02_cfg4_pair_ncu.md (the current kernel, 2e7-path launch; read 129.0 KB, write 0)


def ann_roofline(dims, prec, rate, sl7, peaks, n_sms, sm_max):
    """Roofline of an ANN-mode kernel at `rate` path-steps/s."""
    act = sum(dims[1:-1])
    flops = ann_flops_per_path_step(dims)
    if prec == sl7.PREC_FP32:
        ach = flops * rate / 1e12
        pk = n_sms * 128 * 2 * sm_max * 1e6 / 1e12
        return {"bound": "alu", "pipe": "FP32 FFMA", "achieved": ach, "peak": pk, "unit": "TFLOP/s", "frac": ach / pk,
                "peak_basis": "%d SM x 128 FFMA lanes x 2 FLOP x %g MHz" % (n_sms, sm_max),
                "algorithmic": "%d MLP FLOP per path-step (layer 1 folded to rank 1)" % flops}
    ach = act * rate / 1e12
    pk = n_sms * 16 * sm_max * 1e6 / 1e12
    bf16 = peaks.get("bf16_tflops", 1642.7)
    tpk = bf16 / 2 if prec == sl7.PREC_TF32 else bf16
    mma = (flops - 2 * dims[1]) * rate / 1e12
    r = {"bound": "alu", "pipe": "XU (MUFU)", "achieved": ach, "peak": pk, "unit": "T activations/s", "frac": ach / pk,
         "peak_basis": "%d SM x 16 MUFU op/clk (measured, profiles/r01_pipes.md) x %g MHz" % (n_sms, sm_max),
         "algorithmic": "%d transcendental activations per path-step, counted as ONE MUFU op each" % act,
         "tensor": {"achieved": mma, "peak": tpk, "unit": "TFLOP/s", "frac": mma / tpk,
                    "basis": "%d MMA FLOP per path-step vs MEASURED_PEAKS.json bf16_tflops%s" % (
                        flops - 2 * dims[1], " x 1/2 (tf32:bf16 nominal ratio)" if prec == sl7.PREC_TF32 else "")}}
    if prec in (sl7.PREC_TF32, sl7.PREC_SPLIT):
        # the fp32-class modes need an activation accurate to ~1e-7, which one MUFU op does not give (MUFU.TANH:
        # 1e-5): on the XU pipe alone that is two ops per unit (ex2 + rcp / ex2 + lg2), SURVEY §8(d)'s
        # "accurate" XU bound; the kernels move part of the second op to the FMA pipe
        r["accurate_activation_bound"] = {"ops_per_activation": 2, "peak_path_steps_per_s": pk * 1e12 / (2 * act),
                                          "frac": 2 * ach / pk}
    return r


def run_modes(sl7, torch, dev, stream, peaks, n_sms, sm_max):
    """The other BASELINE configs at N=1 (module docstring), each with its own roofline and clocks."""
    from sl7_inputs import load_golden_blob, workloads
    Wl = workloads()
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device=dev)
    issue_peak = n_sms * 4 * 32 * sm_max * 1e6
    hbm = peaks.get("hbm_gbs", 6454.3)
    out = {}

    def timed(fn, reps=3, warm=1):
        for _ in range(warm):
            fn()
        torch.cuda.synchronize()
        clk = ClockSampler(dev.index)
        clk.start()
        ms = []
        for _ in range(reps):
            flush.fill_(1.0)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            fn()
            e1.record(stream)
            torch.cuda.synchronize()
            ms.append(e0.elapsed_time(e1))
        clk.stop()
        return statistics.mean(ms), clk.summary()

    def issue_roof(rate, instr, what):
        ach = rate * instr
        return {"bound": "alu", "pipe": "issue", "achieved": ach / 1e12, "peak": issue_peak / 1e12,
                "unit": "T thread-instr/s", "frac": ach / issue_peak,
                "algorithmic": "%d instructions per path-step (%s; DESIGN.md §6)" % (instr, what)}

    stats = torch.zeros(sl7.stats_elems(N_BINS), dtype=torch.float64, device=dev)
    P = [("bf16", sl7.PREC_BF16), ("tf32", sl7.PREC_TF32), ("split", sl7.PREC_SPLIT), ("fp32", sl7.PREC_FP32)]

    # ---- cfg3: exact GBM, FULL [65][2e8] fp32 (52 GB) -> HBM store roofline
    w = Wl["cfg3"]
    N, n = w.n_paths, w.n_steps
    buf = torch.empty((n + 1) * N, dtype=torch.float32, device=dev)
    nbytes = 4 * (n + 1) * N
    # store-only HBM peak, measured live: torch fill_ of the same 52 GB buffer (a pure 16-byte store stream)
    fill_ms, _ = timed(lambda: buf.fill_(0.5), reps=3)
    store_peak = nbytes / (fill_ms * 1e-3) / 1e9
    ex = sl7.Context(w.m, device=dev.index)
    for label, flags, instr, what in [
            ("cfg3_exact_gbm_full_specialized", sl7.FLAG_FAST_NORMALS | sl7.FLAG_SPECIALIZED, exact_special_instr(),
             "Philox/4 + fast Box-Muller + closed-form GBM g_m"),
            ("cfg3_exact_gbm_full_general", 0, exact_instr(w.m), "Philox/4 + Box-Muller + barycentric g_m")]:
        o = sl7.make_opts(prec=sl7.PREC_FP32, colloc=sl7.COLLOC_EXACT_GBM, stream=stream, flags=flags)
        ms, clk = timed(lambda o=o: ex.simulate(w.y0, w.dt, n, w.theta, N, w.seed, sl7.OUT_FULL, o, out=buf))
        gbs = nbytes / (ms * 1e-3) / 1e9
        rate = N * n / (ms * 1e-3)
        out[label] = {"path_steps_per_s": rate, "ms": ms, "paths": N, "n_steps": n, "m": w.m,
                      "output": "FULL step-major [65][2e8] fp32, %.1f GB" % (nbytes / 1e9),
                      "roofline": {"bound": "hbm", "achieved": gbs, "peak": hbm, "unit": "GB/s", "frac": gbs / hbm,
                                   "peak_basis": "MEASURED_PEAKS.json hbm_gbs (copy, read+write)",
                                   "store_only_peak": store_peak, "frac_store_only": gbs / store_peak,
                                   "store_only_basis": "torch fill_ of the same buffer, timed here",
                                   "algorithmic": "4 B per path-step + row 0: 4 (n+1) N_P per launch"},
                      "issue_roofline": issue_roof(rate, instr, what), "clocks": clk}
    del buf
    torch.cuda.empty_cache()

    # ---- cfg2: OU (the paper's process) and CIR, 1e8 paths, 16 steps, STATS
    for key in ("cfg2_ou", "cfg2_cir"):
        w = Wl[key]
        ctx = sl7.Context(w.m, list(w.dims), w.act, device=dev.index)
        ctx.load_weights(load_golden_blob(w.blob))
        lo, hi = HIST[w.process]
        N = w.n_paths
        for pn, pc in P:
            n_p = N if pc != sl7.PREC_FP32 else N // 4
            o = sl7.make_opts(prec=pc, colloc=sl7.COLLOC_ANN, stream=stream, n_bins=N_BINS, hist_lo=lo, hist_hi=hi,
                              shift=w.y0)
            ms, clk = timed(lambda o=o, n_p=n_p: ctx.simulate(w.y0, w.dt, w.n_steps, w.theta, n_p, w.seed,
                                                                 sl7.OUT_STATS, o, stats=stats))
            rate = n_p * w.n_steps / (ms * 1e-3)
            s = sl7.stats_summary(stats.cpu().numpy(), o)
            out["%s_%s" % (key, pn)] = {"path_steps_per_s": rate, "ms": ms, "paths": n_p, "n_steps": w.n_steps,
                                        "terminal": {"mean": s["mean"], "var": s["var"]},
                                        "roofline": ann_roofline(w.dims, pc, rate, sl7, peaks, n_sms, sm_max),
                                        "clocks": clk}
        o = sl7.make_opts(prec=sl7.PREC_FP32, colloc=sl7.COLLOC_ANN, scheme=sl7.SCHEME_CDC_PRED, stream=stream,
                          n_bins=N_BINS, hist_lo=lo, hist_hi=hi, shift=w.y0)
        ms, clk = timed(lambda o=o: ctx.simulate(w.y0, w.dt, w.n_steps, w.theta, N, w.seed, sl7.OUT_STATS, o,
                                                 stats=stats))
        rate = N * w.n_steps / (ms * 1e-3)
        s = sl7.stats_summary(stats.cpu().numpy(), o)
        out["%s_cdc_pred" % key] = {"path_steps_per_s": rate, "ms": ms, "paths": N, "n_steps": w.n_steps,
                                    "scheme": "7L-CDC with predicted marginal points (DESIGN.md R-26)",
                                    "terminal": {"mean": s["mean"], "var": s["var"]},
                                    "clamped_path_steps": s.get("clamped_steps"),
                                    "roofline": issue_roof(rate, cdc_pred_instr(w.m),
                                                           "Philox/4 + Box-Muller + clamp + the step as one bivariate "
                                                           "polynomial in (state, X)"),
                                    "frac_vs_lagrange_form_budget": rate * cdc_pred_instr_lagrange(w.m) / issue_peak,
                                    "clocks": clk}
        if w.process == "ou":
            # the same with the fast Box-Muller (SL7_FLAG_FAST_NORMALS, |dX| <= 2e-6 (1 + |X|)), and the quantile-
            # marginal 7L-CDC (R-18: the paper's CDC with the marginal points from all paths' states each step)
            for label, sch, fl in (("cdc_pred_fast_normals", sl7.SCHEME_CDC_PRED, sl7.FLAG_FAST_NORMALS),
                                   ("cdc_quantile", sl7.SCHEME_CDC, 0)):
                o = sl7.make_opts(prec=sl7.PREC_FP32, colloc=sl7.COLLOC_ANN, scheme=sch, stream=stream, flags=fl,
                                  n_bins=N_BINS, hist_lo=lo, hist_hi=hi, shift=w.y0)
                ms, clk = timed(lambda o=o: ctx.simulate(w.y0, w.dt, w.n_steps, w.theta, N, w.seed, sl7.OUT_STATS, o,
                                                         stats=stats))
                rate = N * w.n_steps / (ms * 1e-3)
                s = sl7.stats_summary(stats.cpu().numpy(), o)
                line = {"path_steps_per_s": rate, "ms": ms, "paths": N, "n_steps": w.n_steps,
                        "terminal": {"mean": s["mean"], "var": s["var"]}, "clocks": clk}
                if sch == sl7.SCHEME_CDC_PRED:
                    line["roofline"] = issue_roof(rate, cdc_pred_instr(w.m), "Philox/4 + fast Box-Muller + clamp + "
                                                  "the step as one bivariate polynomial in (state, X)")
                else:
                    line["scheme"] = ("per step: marginal points = exact quantiles of all paths (3 radix-select passes "
                                      "over the states + the pass fused into the step kernel), the m-row table, the step")
                out["%s_%s" % (key, label)] = line
            exo = sl7.Context(w.m, device=dev.index)
            o = sl7.make_opts(prec=sl7.PREC_FP32, colloc=sl7.COLLOC_EXACT_OU, stream=stream, n_bins=N_BINS,
                              hist_lo=lo, hist_hi=hi, shift=w.y0, ref=sl7.REF_OU, ref_theta=w.theta)
            ms, clk = timed(lambda o=o: exo.simulate(w.y0, w.dt, w.n_steps, w.theta, N, w.seed, sl7.OUT_STATS, o,
                                                     stats=stats))
            rate = N * w.n_steps / (ms * 1e-3)
            s = sl7.stats_summary(stats.cpu().numpy(), o)
            out["cfg2_ou_exact"] = {"path_steps_per_s": rate, "ms": ms, "paths": N, "n_steps": w.n_steps,
                                    "terminal": {"mean": s["mean"], "var": s["var"], "strong_err": s["strong_err"]},
                                    "roofline": issue_roof(rate, exact_instr(w.m), "Philox/4 + Box-Muller + g_m + "
                                                           "the Eq. 6.6 reference"), "clocks": clk}

    # ---- cfg4's workload (the headline's) in the other precisions and with CDC_PRED: 1e8 paths (FP32 2.5e7),
    # the same 32 steps to T = 4, terminal moments against the CIR law
    w = Wl["cfg4"]
    ctx = sl7.Context(w.m, list(w.dims), w.act, device=dev.index)
    ctx.load_weights(load_golden_blob(w.blob))
    lo, hi = HIST[w.process]
    for pn, pc in P[1:]:
        n_p = 100_000_000 if pc != sl7.PREC_FP32 else 25_000_000
        o = sl7.make_opts(prec=pc, colloc=sl7.COLLOC_ANN, stream=stream, n_bins=N_BINS, hist_lo=lo, hist_hi=hi,
                          shift=w.y0)
        ms, clk = timed(lambda o=o, n_p=n_p: ctx.simulate(w.y0, w.dt, w.n_steps, w.theta, n_p, w.seed,
                                                             sl7.OUT_STATS, o, stats=stats))
        rate = n_p * w.n_steps / (ms * 1e-3)
        s = sl7.stats_summary(stats.cpu().numpy(), o)
        out["cfg4_%s" % pn] = {"path_steps_per_s": rate, "ms": ms, "paths": n_p, "n_steps": w.n_steps,
                               "terminal": {"mean": s["mean"], "var": s["var"]},
                               "roofline": ann_roofline(w.dims, pc, rate, sl7, peaks, n_sms, sm_max), "clocks": clk}
    o = sl7.make_opts(prec=sl7.PREC_FP32, colloc=sl7.COLLOC_ANN, scheme=sl7.SCHEME_CDC_PRED, stream=stream,
                      n_bins=N_BINS, hist_lo=lo, hist_hi=hi, shift=w.y0)
    ms, clk = timed(lambda o=o: ctx.simulate(w.y0, w.dt, w.n_steps, w.theta, 100_000_000, w.seed, sl7.OUT_STATS, o,
                                             stats=stats))
    rate = 100_000_000 * w.n_steps / (ms * 1e-3)
    s = sl7.stats_summary(stats.cpu().numpy(), o)
    out["cfg4_cdc_pred"] = {"path_steps_per_s": rate, "ms": ms, "paths": 100_000_000, "n_steps": w.n_steps,
                            "scheme": "7L-CDC with predicted marginal points (DESIGN.md R-26)",
                            "terminal": {"mean": s["mean"], "var": s["var"]}, "clamped_path_steps": s.get("clamped_steps"),
                            "roofline": issue_roof(rate, cdc_pred_instr(w.m), "Philox/4 + Box-Muller + clamp + the "
                                                   "step as one bivariate polynomial in (state, X)"), "clocks": clk}
    ctx.close()

    # ---- cfg1: the GBM dt sweep n = 1..64 at 1e7 paths (127 path-steps per path)
    w = Wl["cfg1"]
    N = w.n_paths
    ctx = sl7.Context(w.m, list(w.dims), w.act, device=dev.index)
    ctx.load_weights(load_golden_blob(w.blob))
    ps = N * sum(CFG1_SWEEP)
    for pn, pc in P + [("exact_gbm", None)]:
        c = ctx if pc is not None else sl7.Context(w.m, device=dev.index)
        o = sl7.make_opts(prec=pc if pc is not None else sl7.PREC_FP32,
                          colloc=sl7.COLLOC_ANN if pc is not None else sl7.COLLOC_EXACT_GBM, stream=stream,
                          n_bins=N_BINS, hist_lo=0.0, hist_hi=4.0, shift=1.0, ref=sl7.REF_GBM,
                          ref_theta=(w.theta[0], w.theta[1], 0.0))
        th = () if pc is not None else w.theta
        sts = {ns: torch.zeros(sl7.stats_elems(N_BINS), dtype=torch.float64, device=dev) for ns in CFG1_SWEEP}

        def sweep(c=c, o=o, th=th, sts=sts):
            for ns in CFG1_SWEEP:
                c.simulate(w.y0, 1.0 / ns, ns, th, N, w.seed, sl7.OUT_STATS, o, stats=sts[ns])
        ms, clk = timed(sweep)
        rate = ps / (ms * 1e-3)
        se = {ns: sl7.stats_summary(sts[ns].cpu().numpy(), o)["strong_err"] for ns in CFG1_SWEEP}
        roof = (ann_roofline(w.dims, pc, rate, sl7, peaks, n_sms, sm_max) if pc is not None else
                issue_roof(rate, exact_instr(w.m), "Philox/4 + Box-Muller + g_m + the exact-GBM reference"))
        out["cfg1_sweep_%s" % pn] = {"path_steps_per_s": rate, "ms": ms, "paths": N, "n_sweep": list(CFG1_SWEEP),
                                     "strong_err_by_n": se, "roofline": roof, "clocks": clk}
    return out


if __name__ == "__main__":
    main()
