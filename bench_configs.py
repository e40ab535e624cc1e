"""Per-config measurements beyond bench.py's headline (BASELINE.json configs[2] and [3]), one JSON
line per (config, mode).  Same timing discipline as bench.py: warm-up, L2 flush before each timed
launch, CUDA events on the launch stream, NVML clocks sampled during the timed region.

  python bench_configs.py [--config cfg2|cfg3|all] [--steps K] [--warmup W]

cfg2: OU (Ybar=0, lam=1, sigma=0.5, Y0=1) and CIR (kappa=1, Ybar=0.1, sigma=0.3, Y0=0.1), T=2, 16 steps,
      m=7, [5,50,50,50,50,7] softplus (theta as network input), 1e8 paths, STATS (moments + 4096-bin
      histogram).  Modes: ANN-BF16 (tcgen05), ANN-SPLIT, ANN-FP32, 7L-CDC, exact OU (general / specialised),
      exact CIR (float64 noncentral chi-square quantiles, 1e6 paths).
em:   Euler-Maruyama comparator on cfg2's OU and CIR, 16 large steps of 0.125 with
      K = 1, 8, 125 sub-steps (dtau = 1e-3 at K = 125), STATS + strong error vs the exact OU solution on
      the same fine normals; the 7L lines of cfg2 give the contrast.  Unit: fine path-steps/s.
cfg4: CIR as cfg2, T=4, 32 steps, 4e9 paths in ONE call on one GPU (64-bit path ids past 2^32), STATS;
      ANN-BF16 (tcgen05) and 7L-CDC.  (The scaling runs of BASELINE configs[4] shard these paths over ranks
      with path_offset; only one GPU is available to this harness.)
train: training-set generation (§8(f) row 2): 4096 OU feature rows over SPEC.md:180's ranges
      (dt in [0.05, 2]), M = 1e5 inner paths, dtau = 1e-3 (K_r = ceil(dt/dtau) <= 2000), labels at m = 7.
cfg3: GBM, T=1, 64 steps, m=5, 2e8 paths, FULL step-major path tensor (65 x 2e8 fp32 = 52 GB in HBM).
      Modes: exact GBM with fast normals + closed-form g_m (HBM-store-bound), exact GBM general,
      ANN-BF16 (tcgen05).  Roofline: bound "hbm", algorithmic bytes = 4 (n+1) N_P per launch.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from bench import ClockSampler, measured_peaks  # noqa: E402

UNIT = "path-steps/s"


def timed_launches(fn, steps, warmup, flush, stream):
    import torch
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    ms = []
    for _ in range(steps):
        flush.fill_(1.0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        fn()
        e1.record(stream)
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    return statistics.mean(ms), min(ms)


def _summary(sl7, stats, opts, q_levels=()):
    """stats_summary, or a marker when no terminal value is finite (7L-CDC's polynomial extrapolation into
    the far tails can diverge: DESIGN.md reading R-19) -- the line is still emitted, flagged."""
    try:
        return sl7.stats_summary(stats.cpu().numpy(), opts, q_levels=q_levels)
    except sl7.Sl7Error:
        keys = ("mean", "var", "skew", "exkurt", "strong_err", "rms_err")
        return dict({k: None for k in keys}, n=0, n_nonfinite=int(stats[1].item()), quantiles=None, diverged=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="all", choices=["cfg2", "cfg3", "cfg4", "em", "train", "all"])
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--cfg3-paths", type=int, default=200_000_000)
    ap.add_argument("--cfg2-paths", type=int, default=100_000_000)
    ap.add_argument("--cfg4-paths", type=int, default=4_000_000_000)
    ap.add_argument("--train-rows", type=int, default=4096)
    ap.add_argument("--train-inner", type=int, default=100_000)
    a = ap.parse_args()

    import torch
    import paper_2302_05170_b200 as sl7
    from sl7_inputs import load_golden_blob, workloads
    sl7.load_library()
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    stream = torch.cuda.current_stream()
    flush = torch.empty((512 << 20) // 4, dtype=torch.float32, device=dev)
    peaks = measured_peaks()
    hbm = peaks.get("hbm_gbs", 6454.3)
    sm_max = peaks.get("sm_max_mhz", 1965.0)
    n_sms = torch.cuda.get_device_properties(dev).multi_processor_count
    Wl = workloads()

    def emit(d):
        # a run with non-finite terminal values (7L-CDC with quantile marginals on CIR diverges, R-25)
        # has no throughput: its value is withheld and the line says why
        t = d.get("terminal") or {}
        nnf = d.get("n_nonfinite", 0)
        if d.get("value") is not None and (t.get("mean") is None or (nnf or 0) > 0) and "terminal" in d:
            d = dict(d, value=None, diverged=True, rate_withheld="non-finite terminal values: no valid throughput")
            d.pop("roofline", None)
        print(json.dumps(d), flush=True)

    if a.config in ("cfg3", "all"):
        w = Wl["cfg3"]
        N, n = a.cfg3_paths, w.n_steps
        out = torch.empty((n + 1) * N, dtype=torch.float32, device=dev)
        bytes_per_launch = 4 * (n + 1) * N
        ctx_ex = sl7.Context(w.m, device=0)
        ctx_ann = sl7.Context(w.m, list(w.dims), w.act, device=0)
        ctx_ann.load_weights(load_golden_blob(w.blob))
        modes = [("exact_gbm_fast_specialized", ctx_ex, sl7.COLLOC_EXACT_GBM, sl7.PREC_FP32,
                  sl7.FLAG_FAST_NORMALS | sl7.FLAG_SPECIALIZED, w.theta),
                 ("exact_gbm_general", ctx_ex, sl7.COLLOC_EXACT_GBM, sl7.PREC_FP32, 0, w.theta),
                 ("ann_bf16_tcgen05", ctx_ann, sl7.COLLOC_ANN, sl7.PREC_BF16, 0, ())]
        for label, ctx, colloc, prec, flags, theta in modes:
            opts = sl7.make_opts(prec=prec, colloc=colloc, stream=stream, flags=flags)
            fn = (lambda ctx=ctx, theta=theta, opts=opts:
                  ctx.simulate(w.y0, w.dt, n, theta, N, w.seed, sl7.OUT_FULL, opts, out=out))
            clk = ClockSampler(0)
            clk.start()
            ms, ms_min = timed_launches(fn, a.steps, a.warmup, flush, stream)
            clk.stop()
            gbs = bytes_per_launch / (ms * 1e-3) / 1e9
            emit({"config": "cfg3", "mode": label, "metric": "7L path-steps/sec (device-timed)",
                  "value": N * n / (ms * 1e-3), "unit": UNIT, "ms_per_launch": ms, "ms_min": ms_min,
                  "paths": N, "n_steps": n, "m": w.m, "output": "FULL step-major [65][N] fp32 (%.1f GB)" % (bytes_per_launch / 1e9),
                  "roofline": {"bound": "hbm", "achieved": gbs, "peak": hbm, "unit": "GB/s", "frac": gbs / hbm,
                               "traffic": None, "algorithmic": "4 B per path-step + row 0 (4 (n+1) N_P per launch)",
                               "peak_basis": "MEASURED_PEAKS.json hbm_gbs (copy, read+write)"},
                  "clocks": clk.summary()})
        del out
        torch.cuda.empty_cache()

    # issue roofline of the RNG-bound kernels: thread-instructions/s = SMs x 4 schedulers x 32 lanes x clock,
    # against an ALGORITHMIC instruction budget per (fine) path-step, not the kernel's own SASS count
    # (bench.py's budgets): EM = Philox4x32-10 / 4 normals (11) + Box-Muller (9) + the
    # Euler update (3: drift FFMA, diffusion FFMA, the CIR truncation or the GBM product)
    from bench import BOX_MULLER_PER_NORMAL, PHILOX_PER_NORMAL, cdc_pred_instr
    issue_peak = n_sms * 4 * 32 * sm_max * 1e6
    em_instr = float(PHILOX_PER_NORMAL + BOX_MULLER_PER_NORMAL + 3)

    if a.config in ("em", "all"):
        from sl7_inputs import CIR_THETA, OU_THETA
        stats = torch.zeros(sl7.stats_elems(4096), dtype=torch.float64, device=dev)
        ctx = sl7.Context(7, device=0)
        for proc, theta, y0, model, lo, hi in [("ou", OU_THETA, 1.0, sl7.MODEL_OU, -3.0, 3.0),
                                               ("cir", CIR_THETA, 0.1, sl7.MODEL_CIR, 0.0, 0.6)]:
            for K, N in [(1, 100_000_000), (8, 25_000_000), (125, 2_000_000)]:
                for fast in (False, True):
                    flags = sl7.FLAG_FAST_NORMALS if fast else 0
                    ref = sl7.REF_OU if proc == "ou" else sl7.REF_NONE
                    opts = sl7.make_opts(stream=stream, n_bins=4096, hist_lo=lo, hist_hi=hi, shift=y0, ref=ref,
                                         ref_theta=theta, flags=flags)
                    fn = (lambda opts=opts, K=K, N=N, model=model, theta=theta, y0=y0:
                          ctx.simulate_em(model, y0, 0.125, 16, K, theta, N, 2302051702, sl7.OUT_STATS, opts,
                                          stats=stats))
                    clk = ClockSampler(0)
                    clk.start()
                    ms, ms_min = timed_launches(fn, a.steps, a.warmup, flush, stream)
                    clk.stop()
                    s = _summary(sl7, stats, opts)
                    rate = N * 16 * K / (ms * 1e-3)
                    line = {"config": "em_" + proc, "mode": "euler_maruyama_K%d%s" % (K, "_fast" if fast else ""),
                            "metric": "Euler-Maruyama fine path-steps/sec (device-timed)", "value": rate,
                            "unit": "fine path-steps/s", "ms_per_launch": ms, "paths": N, "n_steps": 16,
                            "substeps": K, "dtau": 0.125 / K,
                            "terminal": {k: s[k] for k in ("mean", "var", "strong_err")}, "clocks": clk.summary()}
                    if fast:
                        ach = rate * em_instr
                        line["roofline"] = {"bound": "alu", "pipe": "issue", "achieved": ach / 1e12,
                                            "peak": issue_peak / 1e12, "unit": "T thread-instr/s",
                                            "frac": ach / issue_peak,
                                            "algorithmic": "%.0f instructions per fine path-step" % em_instr}
                    emit(line)

    if a.config in ("train", "all"):
        import numpy as np
        from sl7_inputs import sample_features
        R, M, dtau, m = a.train_rows, a.train_inner, 1e-3, 7
        F = sample_features("ou", R, seed=2302051705)
        K = np.maximum(1, np.ceil(F[:, 1] / dtau))
        fine = float(K.sum()) * M
        ctx = sl7.Context(m, device=0)
        labels = torch.empty((R, m), dtype=torch.float64, device=dev)
        for fast in (False, True):
            opts = sl7.make_opts(stream=stream, flags=sl7.FLAG_FAST_NORMALS if fast else 0)
            fn = (lambda opts=opts: ctx.training_set(sl7.MODEL_OU, F, M, dtau, 2302051705, opts, labels=labels))
            clk = ClockSampler(0)
            clk.start()
            ms, ms_min = timed_launches(fn, a.steps, a.warmup, flush, stream)
            clk.stop()
            rate = fine / (ms * 1e-3)
            line = {"config": "train_ou", "mode": "training_set%s" % ("_fast" if fast else ""),
                    "metric": "training rows/sec (device-timed)", "value": R / (ms * 1e-3), "unit": "rows/s",
                    "fine_path_steps_per_s": rate, "ms_per_launch": ms, "rows": R, "inner_paths": M, "dtau": dtau,
                    "mean_substeps": float(K.mean()), "m": m, "clocks": clk.summary()}
            if fast:
                ach = rate * em_instr
                line["roofline"] = {"bound": "alu", "pipe": "issue", "achieved": ach / 1e12, "peak": issue_peak / 1e12,
                                    "unit": "T thread-instr/s", "frac": ach / issue_peak,
                                    "algorithmic": "%.0f instructions per fine path-step" % em_instr}
            emit(line)

    if a.config in ("cfg4", "all"):
        w = Wl["cfg4"]
        N = a.cfg4_paths
        stats = torch.zeros(sl7.stats_elems(4096), dtype=torch.float64, device=dev)
        ctx = sl7.Context(w.m, list(w.dims), w.act, device=0)
        ctx.load_weights(load_golden_blob(w.blob))
        for label, prec, scheme, n_paths in [("ann_bf16_tcgen05", sl7.PREC_BF16, sl7.SCHEME_7L, N),
                                             ("cdc_pred_ann_fp32_table", sl7.PREC_FP32, sl7.SCHEME_CDC_PRED, N // 10),
                                             ("cdc_ann_fp32_table", sl7.PREC_FP32, sl7.SCHEME_CDC, N // 10)]:
            opts = sl7.make_opts(prec=prec, colloc=sl7.COLLOC_ANN, stream=stream, n_bins=4096, hist_lo=0.0, hist_hi=0.6,
                                 shift=w.y0, scheme=scheme)
            fn = (lambda opts=opts, n_paths=n_paths:
                  ctx.simulate(w.y0, w.dt, w.n_steps, w.theta, n_paths, w.seed, sl7.OUT_STATS, opts, stats=stats))
            clk = ClockSampler(0)
            clk.start()
            ms, ms_min = timed_launches(fn, max(1, a.steps - 1), 1, flush, stream)
            clk.stop()
            s = _summary(sl7, stats, opts, [0.01, 0.5, 0.99])
            rate = n_paths * w.n_steps / (ms * 1e-3)
            line = {"config": "cfg4", "mode": label, "metric": "7L path-steps/sec (device-timed)", "value": rate,
                    "unit": UNIT, "ms_per_launch": ms, "paths": n_paths, "n_steps": w.n_steps, "m": w.m,
                    "terminal": {k: s[k] for k in ("mean", "var", "skew", "exkurt")}, "n_counted": s["n"],
                    "n_nonfinite": s["n_nonfinite"], "quantiles_1_50_99": s["quantiles"], "clocks": clk.summary()}
            if prec == sl7.PREC_BF16:
                trans = sum(w.dims[1:-1])
                ach = trans * rate / 1e12
                pk = n_sms * 16 * sm_max * 1e6 / 1e12
                line["roofline"] = {"bound": "alu", "pipe": "XU (MUFU)", "achieved": ach, "peak": pk, "unit": "Top/s",
                                    "frac": ach / pk, "algorithmic": "%d softplus activations per path-step" % trans}
            emit(line)

    if a.config in ("cfg2", "all"):
        N = a.cfg2_paths
        stats = torch.zeros(sl7.stats_elems(4096), dtype=torch.float64, device=dev)
        for key in ("cfg2_ou", "cfg2_cir"):
            w = Wl[key]
            ctx = sl7.Context(w.m, list(w.dims), w.act, device=0)
            ctx.load_weights(load_golden_blob(w.blob))
            lo, hi = (-3.0, 3.0) if w.process == "ou" else (0.0, 0.6)
            modes = [("ann_bf16_tcgen05", ctx, sl7.COLLOC_ANN, sl7.PREC_BF16, 0, w.theta, N),
                     ("ann_tf32_tcgen05", ctx, sl7.COLLOC_ANN, sl7.PREC_TF32, 0, w.theta, N),
                     ("ann_split_bf16x3_tcgen05", ctx, sl7.COLLOC_ANN, sl7.PREC_SPLIT, 0, w.theta, N),
                     ("ann_fp32", ctx, sl7.COLLOC_ANN, sl7.PREC_FP32, 0, w.theta, N // 10),
                     ("cdc_ann_fp32_table", ctx, sl7.COLLOC_ANN, sl7.PREC_FP32, -1, w.theta, N),
                     ("cdc_ann_fp32_table_fast_normals", ctx, sl7.COLLOC_ANN, sl7.PREC_FP32, -2, w.theta, N),
                     ("cdc_pred_ann_fp32_table", ctx, sl7.COLLOC_ANN, sl7.PREC_FP32, -3, w.theta, N),
                     ("cdc_pred_ann_fp32_table_fast_normals", ctx, sl7.COLLOC_ANN, sl7.PREC_FP32, -4, w.theta, N)]
            if w.process == "cir":
                ex = sl7.Context(w.m, device=0)
                modes += [("exact_cir_ncx2_fp64", ex, sl7.COLLOC_EXACT_CIR, sl7.PREC_FP32, 0, w.theta, N // 100)]
            if w.process == "ou":
                ex = sl7.Context(w.m, device=0)
                modes += [("exact_ou_general", ex, sl7.COLLOC_EXACT_OU, sl7.PREC_FP32, 0, w.theta, N),
                          ("exact_ou_fast_specialized", ex, sl7.COLLOC_EXACT_OU, sl7.PREC_FP32,
                           sl7.FLAG_FAST_NORMALS | sl7.FLAG_SPECIALIZED, w.theta, N)]
            for label, c, colloc, prec, flags, theta, n_paths in modes:
                # markers: 7L-CDC scheme (-1, -2) or CDC_PRED (-3, -4); -2, -4 with SL7_FLAG_FAST_NORMALS
                cdc = flags < 0
                scheme = (sl7.SCHEME_CDC if flags in (-1, -2) else sl7.SCHEME_CDC_PRED) if cdc else sl7.SCHEME_7L
                ref = sl7.REF_OU if (w.process == "ou" and not cdc) else sl7.REF_NONE
                fl = (sl7.FLAG_FAST_NORMALS if flags in (-2, -4) else 0) if cdc else flags
                opts = sl7.make_opts(prec=prec, colloc=colloc, stream=stream, flags=fl, n_bins=4096,
                                     hist_lo=lo, hist_hi=hi, shift=w.y0, ref=ref, ref_theta=w.theta,
                                     scheme=scheme)
                fn = (lambda c=c, theta=theta, opts=opts, n_paths=n_paths:
                      c.simulate(w.y0, w.dt, w.n_steps, theta, n_paths, w.seed, sl7.OUT_STATS, opts, stats=stats))
                clk = ClockSampler(0)
                clk.start()
                ms, ms_min = timed_launches(fn, a.steps, a.warmup, flush, stream)
                clk.stop()
                s = _summary(sl7, stats, opts, [0.01, 0.5, 0.99])
                rate = n_paths * w.n_steps / (ms * 1e-3)
                line = {"config": key, "mode": label, "metric": "7L path-steps/sec (device-timed)", "value": rate,
                        "unit": UNIT, "ms_per_launch": ms, "paths": n_paths, "n_steps": w.n_steps, "m": w.m,
                        "terminal": {k: s[k] for k in ("mean", "var", "skew", "exkurt", "strong_err")},
                        "quantiles_1_50_99": s["quantiles"], "clocks": clk.summary()}
                if flags == -3:
                    # fused CDC_PRED kernel: issue-bound; algorithmic budget (bench.cdc_pred_instr): Philox/4 +
                    # Box-Muller + clamp + the step as one bivariate polynomial (m(m-1) + m-1 FMA)
                    instr = cdc_pred_instr(w.m)
                    ach = rate * instr
                    line["roofline"] = {"bound": "alu", "pipe": "issue", "achieved": ach / 1e12,
                                        "peak": issue_peak / 1e12, "unit": "T thread-instr/s", "frac": ach / issue_peak,
                                        "algorithmic": "%d instructions per path-step (algorithmic budget)" % instr}
                if colloc == sl7.COLLOC_ANN and prec in (sl7.PREC_BF16, sl7.PREC_TF32):
                    trans = sum(w.dims[1:-1])
                    ach = trans * rate / 1e12
                    pk = n_sms * 16 * sm_max * 1e6 / 1e12
                    line["roofline"] = {"bound": "alu", "pipe": "XU (MUFU)", "achieved": ach, "peak": pk,
                                        "unit": "Top/s", "frac": ach / pk,
                                        "algorithmic": "%d softplus activations per path-step" % trans}
                emit(line)
            # the sharded-CDC driver (sl7_cdc_* + dist.cdc_run) on one rank: the cost of driving the per-pass
            # exchange from the host, against the single-call CDC line above
            from paper_2302_05170_b200.dist import CdcShard, cdc_run
            opts = sl7.make_opts(prec=sl7.PREC_FP32, colloc=sl7.COLLOC_ANN, stream=stream, n_bins=4096, hist_lo=lo,
                                 hist_hi=hi, shift=w.y0, scheme=sl7.SCHEME_CDC)

            def sharded(opts=opts, ctx=ctx, w=w):
                stats.zero_()
                cdc_run([CdcShard(ctx, w.y0, w.dt, w.n_steps, w.theta, N, w.seed, opts, stats)], w.n_steps,
                        allreduce=lambda t: None)
            clk = ClockSampler(0)
            clk.start()
            ms, ms_min = timed_launches(sharded, a.steps, a.warmup, flush, stream)
            clk.stop()
            s = _summary(sl7, stats, opts, [0.01, 0.5, 0.99])
            emit({"config": key, "mode": "cdc_sharded_driver_1rank", "metric": "7L path-steps/sec (device-timed)",
                  "value": N * w.n_steps / (ms * 1e-3), "unit": UNIT, "ms_per_launch": ms, "paths": N,
                  "n_steps": w.n_steps, "m": w.m, "exchange": "4 x %d-byte histogram all-reduces per step" % (
                      8 * sl7.cdc_hist_elems()),
                  "terminal": {k: s[k] for k in ("mean", "var", "skew", "exkurt", "strong_err")},
                  "clocks": clk.summary()})


if __name__ == "__main__":
    main()
