"""C-ABI behaviour on the GPU: argument validation, chunked (resumed) runs, host-buffer entry point,
degenerate sizes for every kernel family."""
import numpy as np
import pytest

from oracle import sl7_oracle as O
from sl7_inputs import load_golden_blob, workloads

pytestmark = pytest.mark.gpu


def _torch():
    import torch
    return torch


def test_validation_errors(gpu_lib):
    sl7 = gpu_lib
    torch = _torch()
    ctx = sl7.Context(5)
    out = torch.empty(10, dtype=torch.float32, device="cuda")
    st = torch.zeros(sl7.stats_elems(8), dtype=torch.float64, device="cuda")

    def call(dt=0.5, n_steps=2, n_paths=10, theta=(0.05, 0.2), mode=None, **kw):
        o = sl7.make_opts(colloc=sl7.COLLOC_EXACT_GBM, **kw)
        return ctx.simulate(1.0, dt, n_steps, theta, n_paths, 1, sl7.OUT_TERMINAL if mode is None else mode, o,
                            out=out, stats=st)

    for kw, msg in [(dict(dt=0.0), "dt"), (dict(dt=float("nan")), "dt"), (dict(n_steps=0), "n_steps"),
                    (dict(n_paths=0), "n_paths"), (dict(theta=(0.05,)), "EXACT_GBM"),
                    (dict(theta=(0.05, -0.2)), "sigma"), (dict(n_bins=20000, hist_lo=0, hist_hi=1), "n_bins"),
                    (dict(n_bins=8, hist_lo=1, hist_hi=1), "hist_lo"), (dict(flags=8), "flags"),
                    (dict(scheme=5), "scheme"), (dict(path_offset=(1 << 64) - 5), "overflows")]:
        with pytest.raises(sl7.Sl7Error, match=msg):
            call(**kw)
    import ctypes
    th = (ctypes.c_double * 2)(0.05, 0.2)
    o = sl7.make_opts(colloc=sl7.COLLOC_EXACT_GBM)
    st_ = sl7._lib.sl7_simulate(ctx._h, 1.0, 0.5, 2, th, 2, 10, 1, sl7.OUT_FULL, ctypes.byref(o), None, None)
    assert st_ == sl7.EINVAL and b"d_out" in sl7._lib.sl7_last_error(ctx._h)
    with pytest.raises(sl7.Sl7Error, match="ESTATE"):
        ctx.simulate(1.0, 0.5, 2, (), 10, 1, sl7.OUT_TERMINAL, sl7.make_opts(colloc=sl7.COLLOC_ANN), out=out)


@pytest.mark.parametrize("prec", ["fp32", "bf16", "tf32", "split"])
def test_chunked_accumulate_equals_single_run(gpu_lib, prec):
    """Checkpoint/resume semantics: the counter-based RNG makes any path range recomputable, and
    opts.accumulate sums chunk statistics into one vector."""
    sl7 = gpu_lib
    torch = _torch()
    p = {"fp32": sl7.PREC_FP32, "bf16": sl7.PREC_BF16, "tf32": sl7.PREC_TF32, "split": sl7.PREC_SPLIT}[prec]
    w = workloads()["cfg2_ou"]
    ctx = sl7.Context(w.m, list(w.dims), w.act)
    ctx.load_weights(load_golden_blob(w.blob))
    N = 40_001
    kw = dict(prec=p, colloc=sl7.COLLOC_ANN, n_bins=256, hist_lo=-3, hist_hi=3, shift=0.0)
    full = torch.zeros(sl7.stats_elems(256), dtype=torch.float64, device="cuda")
    ctx.simulate(w.y0, w.dt, 8, w.theta, N, 7, sl7.OUT_STATS, sl7.make_opts(**kw), stats=full)
    acc = torch.zeros_like(full)
    for lo, n in [(0, 10_000), (10_000, 1), (10_001, 30_000)]:
        ctx.simulate(w.y0, w.dt, 8, w.theta, n, 7, sl7.OUT_STATS, sl7.make_opts(path_offset=lo, accumulate=1, **kw),
                     stats=acc)
    torch.cuda.synchronize()
    a, f = acc.cpu().numpy(), full.cpu().numpy()
    assert a[0] == f[0] == N and np.array_equal(a[8:], f[8:])
    np.testing.assert_allclose(a[2:6], f[2:6], rtol=1e-12)


def test_host_entry_stats_only(gpu_lib):
    sl7 = gpu_lib
    torch = _torch()
    ctx = sl7.Context(7)
    opts = sl7.make_opts(colloc=sl7.COLLOC_EXACT_OU, n_bins=64, hist_lo=-2, hist_hi=3, shift=1.0,
                         ref=sl7.REF_OU, ref_theta=(0.0, 1.0, 0.5))
    h = np.empty(sl7.stats_elems(64))
    _, _, up, down = ctx.simulate_host(1.0, 0.125, 16, (0.0, 1.0, 0.5), 100_000, 3, sl7.OUT_STATS, opts, None, h)
    d = torch.zeros(sl7.stats_elems(64), dtype=torch.float64, device="cuda")
    ctx.simulate(1.0, 0.125, 16, (0.0, 1.0, 0.5), 100_000, 3, sl7.OUT_STATS, opts, stats=d)
    torch.cuda.synchronize()
    np.testing.assert_allclose(h, d.cpu().numpy(), rtol=1e-12)
    assert down == h.nbytes and h[0] == 100_000
    s = sl7.stats_summary(h, opts)
    assert s["strong_err"] < 1e-6      # exact OU collocation = Eq. 6.6 on the same normals


@pytest.mark.parametrize("kind", ["exact", "fp32", "bf16", "tf32", "split", "cdc"])
def test_single_path_and_single_step(gpu_lib, kind):
    sl7 = gpu_lib
    torch = _torch()
    w = workloads()["cfg0"]
    blob = load_golden_blob(w.blob)
    if kind == "exact":
        ctx, colloc, theta, prec = sl7.Context(5), sl7.COLLOC_EXACT_GBM, w.theta, sl7.PREC_FP32
    else:
        ctx = sl7.Context(w.m, list(w.dims), w.act)
        ctx.load_weights(blob)
        colloc, theta = sl7.COLLOC_ANN, ()
        prec = {"fp32": sl7.PREC_FP32, "bf16": sl7.PREC_BF16, "tf32": sl7.PREC_TF32, "split": sl7.PREC_SPLIT,
                "cdc": sl7.PREC_FP32}[kind]
    scheme = sl7.SCHEME_CDC if kind == "cdc" else sl7.SCHEME_7L
    for n_paths, n_steps in [(1, 1), (1, 5), (129, 1)]:
        o = sl7.make_opts(prec=prec, colloc=colloc, scheme=scheme)
        out, _ = ctx.simulate(1.0, 0.5, n_steps, theta, n_paths, 5, sl7.OUT_FULL, o)
        torch.cuda.synchronize()
        Yd = out.double().cpu().numpy().reshape(n_steps + 1, n_paths)
        spec = O.Spec(5, "gbm" if kind == "exact" else "ann", theta, 1.0, 0.5, n_steps, net=O.parse_blob(blob),
                      quant=kind if kind in ("bf16", "tf32") else None)
        Z = O.normals(5, np.arange(n_paths, dtype=np.uint64), n_steps)
        tol = 5e-3 if kind in ("bf16", "tf32") else 1e-5
        for i in range(n_steps):
            if kind == "cdc":
                ref, kap = O.cdc_step(spec, Yd[i], Z[i]), O.cdc_step_error_scale(spec, Yd[i], Z[i])
            else:
                ref, kap = O.step(spec, Yd[i], Z[i]), O.step_error_scale(spec, Yd[i], Z[i])
            assert np.all(np.abs(Yd[i + 1] - ref) <= tol * kap), (kind, n_paths, n_steps, i)


@pytest.mark.parametrize("kind", ["exact", "fp32", "bf16", "tf32", "split", "cdc", "em"])
def test_max_histogram_bins(gpu_lib, kind):
    """The largest histogram (16384 bins, 64 KB of shared memory next to the weight tiles and, in the
    tensor-core kernels, the per-thread statistics) on the deepest network (cfg2, 4 hidden layers): the
    fused histogram equals numpy's histogram of the same run's terminal values, count for count."""
    sl7 = gpu_lib
    torch = _torch()
    w = workloads()["cfg2_ou"]
    nb, lo, hi, N = 16384, -3.0, 3.0, 50_000
    st = torch.zeros(sl7.stats_elems(nb), dtype=torch.float64, device="cuda")
    kw = dict(n_bins=nb, hist_lo=lo, hist_hi=hi, shift=1.0)
    if kind in ("exact", "em"):
        ctx = sl7.Context(w.m)
    else:
        ctx = sl7.Context(w.m, list(w.dims), w.act)
        ctx.load_weights(load_golden_blob(w.blob))
    if kind == "em":
        out, _ = ctx.simulate_em(sl7.MODEL_OU, w.y0, w.dt, w.n_steps, 2, w.theta, N, w.seed, sl7.OUT_TERMINAL,
                                 sl7.make_opts(**kw), stats=st)
    else:
        colloc = sl7.COLLOC_EXACT_OU if kind == "exact" else sl7.COLLOC_ANN
        prec = {"exact": sl7.PREC_FP32, "fp32": sl7.PREC_FP32, "bf16": sl7.PREC_BF16, "tf32": sl7.PREC_TF32,
                "split": sl7.PREC_SPLIT, "cdc": sl7.PREC_FP32}[kind]
        scheme = sl7.SCHEME_CDC if kind == "cdc" else sl7.SCHEME_7L
        out, _ = ctx.simulate(w.y0, w.dt, w.n_steps, w.theta, N, w.seed, sl7.OUT_TERMINAL,
                              sl7.make_opts(prec=prec, colloc=colloc, scheme=scheme, **kw), stats=st)
    torch.cuda.synchronize()
    v = st.cpu().numpy()
    ref = O.stats_vector(out.double().cpu().numpy(), 1.0, lo, hi, nb)
    assert v[0] == ref[0] == N
    np.testing.assert_array_equal(v[8:], ref[8:])
    np.testing.assert_allclose(v[2:6], ref[2:6], rtol=1e-10)


def test_binding_rejects_undersized_or_mistyped_buffers(gpu_lib):
    """The C ABI takes plain device pointers; the binding checks dtype, device, contiguity and size first."""
    sl7 = gpu_lib
    torch = _torch()
    ctx = sl7.Context(5)
    o = sl7.make_opts(colloc=sl7.COLLOC_EXACT_GBM)
    th = (0.05, 0.2)
    for out, msg in [(torch.empty(29, dtype=torch.float32, device="cuda"), "needed"),
                     (torch.empty(30, dtype=torch.float64, device="cuda"), "float32"),
                     (torch.empty(30, dtype=torch.float32), "CUDA"),
                     (torch.empty(60, dtype=torch.float32, device="cuda")[::2], "contiguous")]:
        with pytest.raises(sl7.Sl7Error, match=msg):
            ctx.simulate(1.0, 0.5, 2, th, 10, 1, sl7.OUT_FULL, o, out=out)
    with pytest.raises(sl7.Sl7Error, match="stats"):
        ctx.simulate(1.0, 0.5, 2, th, 10, 1, sl7.OUT_STATS, sl7.make_opts(colloc=sl7.COLLOC_EXACT_GBM, n_bins=64,
                                                                          hist_lo=0, hist_hi=2),
                     stats=torch.zeros(sl7.stats_elems(64) - 1, dtype=torch.float64, device="cuda"))
    with pytest.raises(sl7.Sl7Error, match="h_out"):
        ctx.simulate_host(1.0, 0.5, 2, th, 10, 1, sl7.OUT_TERMINAL, o, np.empty(9, dtype=np.float32))


def test_host_async_pipeline_equals_sync_calls(gpu_lib):
    """Several sl7_simulate_host_async calls in flight (two staging slots, copies overlapping the next
    call's kernels) give exactly the results of the blocking calls."""
    sl7 = gpu_lib
    torch = _torch()
    w = workloads()["cfg1"]
    ctx = sl7.Context(w.m, list(w.dims), w.act)
    ctx.load_weights(load_golden_blob(w.blob))
    opts = sl7.make_opts(prec=sl7.PREC_BF16, colloc=sl7.COLLOC_ANN, n_bins=64, hist_lo=0, hist_hi=4, shift=1.0)
    N, sweep = 300_001, (1, 2, 4, 8, 16)
    outs = [torch.empty(N, dtype=torch.float32, pin_memory=True).numpy() for _ in sweep]
    sts = [torch.empty(sl7.stats_elems(64), dtype=torch.float64, pin_memory=True).numpy() for _ in sweep]
    for ns, o, s_ in zip(sweep, outs, sts):
        ctx.simulate_host_async(w.y0, 1.0 / ns, ns, (), N, w.seed, sl7.OUT_TERMINAL, opts, o, s_)
    ctx.sync()
    for ns, o, s_ in zip(sweep, outs, sts):
        ro = np.empty(N, dtype=np.float32)
        rs = np.empty(sl7.stats_elems(64), dtype=np.float64)
        ctx.simulate_host(w.y0, 1.0 / ns, ns, (), N, w.seed, sl7.OUT_TERMINAL, opts, ro, rs)
        np.testing.assert_array_equal(o, ro)
        assert s_[0] == rs[0] == N and np.array_equal(s_[8:], rs[8:])
        np.testing.assert_allclose(s_[2:6], rs[2:6], rtol=1e-12)


def test_nonfinite_paths_are_counted_not_summed(gpu_lib):
    """Paths that overflow (GBM with an absurd volatility) are counted in n_nonfinite and left out of the
    sums and the histogram; the host summary then reports SL7_ENONFINITE."""
    sl7 = gpu_lib
    torch = _torch()
    ctx = sl7.Context(5)
    N = 4096
    st = torch.zeros(sl7.stats_elems(16), dtype=torch.float64, device="cuda")
    opts = sl7.make_opts(colloc=sl7.COLLOC_EXACT_GBM, n_bins=16, hist_lo=0.0, hist_hi=10.0)
    out, _ = ctx.simulate(1.0, 1.0, 47, (2.0, 0.5), N, 2, sl7.OUT_TERMINAL, opts, stats=st)   # log Y_T ~ N(88, 3.4^2)
    torch.cuda.synchronize()
    Y = out.double().cpu().numpy()
    v = st.cpu().numpy()
    fin = np.isfinite(Y)
    assert 0 < (~fin).sum() < N
    assert v[0] == fin.sum() and v[1] == (~fin).sum()
    ref = O.stats_vector(Y, 0.0, 0.0, 10.0, 16)
    np.testing.assert_array_equal(v[8:], ref[8:])
    s = sl7.stats_summary(v, opts)
    assert s["status"] == sl7.ENONFINITE and s["n_nonfinite"] == (~fin).sum()


@pytest.mark.parametrize("mode", ["ann_bf16", "ann_fp32", "cdc", "em"])
def test_side_stream_equals_default_stream(gpu_lib, mode):
    """opts.stream is honoured: every kernel family enqueued on a side stream (with the output buffers
    allocated on it) gives bitwise the default-stream result once that stream is synchronised."""
    sl7 = gpu_lib
    torch = _torch()
    w = workloads()["cfg2_ou"]
    n, steps = 40_003, 6

    def run(stream):
        ctx = sl7.Context(w.m, list(w.dims), w.act)
        ctx.load_weights(load_golden_blob(w.blob))
        kw = dict(stream=stream, n_bins=256, hist_lo=-3.0, hist_hi=3.0)
        if mode == "em":
            opts = sl7.make_opts(**kw)
            out, st = ctx.simulate_em(sl7.MODEL_OU, w.y0, w.dt, steps, 4, w.theta, n, w.seed, sl7.OUT_TERMINAL, opts,
                                      stats=torch.zeros(sl7.stats_elems(256), dtype=torch.float64, device="cuda"))
        else:
            prec = sl7.PREC_BF16 if mode == "ann_bf16" else sl7.PREC_FP32
            scheme = sl7.SCHEME_CDC if mode == "cdc" else sl7.SCHEME_7L
            opts = sl7.make_opts(prec=prec, colloc=sl7.COLLOC_ANN, scheme=scheme, **kw)
            out, st = ctx.simulate(w.y0, w.dt, steps, w.theta, n, w.seed, sl7.OUT_TERMINAL, opts,
                                   stats=torch.zeros(sl7.stats_elems(256), dtype=torch.float64, device="cuda"))
        return ctx, out, st

    _, ref_out, ref_st = run(None)
    torch.cuda.synchronize()
    ref_out, ref_st = ref_out.clone(), ref_st.clone()
    side = torch.cuda.Stream()
    with torch.cuda.stream(side):
        ctx, out, st = run(side)
        ev = torch.cuda.Event()
        ev.record(side)
    side.synchronize()
    assert ev.query()
    assert torch.equal(out, ref_out)
    torch.testing.assert_close(st[:2], ref_st[:2], rtol=0, atol=0)          # counts
    torch.testing.assert_close(st[8:], ref_st[8:], rtol=0, atol=0)          # histogram
    torch.testing.assert_close(st, ref_st, rtol=1e-12, atol=0)              # fp64 sums (atomic order)


def test_contexts_release_their_device_memory(gpu_lib):
    """Creating, using (every buffer-owning path: weights, 7L-CDC scratch and state, the pipelined host API's
    staging slots and copy stream) and closing contexts in a loop leaves the device's free memory where it
    was: sl7_destroy frees everything the context allocated."""
    sl7 = gpu_lib
    torch = _torch()
    w = workloads()["cfg2_ou"]
    blob = load_golden_blob(w.blob)
    n = 200_000

    def cycle():
        with sl7.Context(w.m, list(w.dims), w.act) as ctx:
            ctx.load_weights(blob)
            st = torch.zeros(sl7.stats_elems(64), dtype=torch.float64, device="cuda")
            kw = dict(n_bins=64, hist_lo=-3.0, hist_hi=3.0)
            for prec in (sl7.PREC_BF16, sl7.PREC_FP32):
                ctx.simulate(w.y0, w.dt, 4, w.theta, n, 1, sl7.OUT_STATS,
                             sl7.make_opts(prec=prec, colloc=sl7.COLLOC_ANN, **kw), stats=st)
            ctx.simulate(w.y0, w.dt, 4, w.theta, n, 1, sl7.OUT_STATS,
                         sl7.make_opts(colloc=sl7.COLLOC_ANN, scheme=sl7.SCHEME_CDC, **kw), stats=st)
            ctx.simulate_em(sl7.MODEL_OU, w.y0, w.dt, 4, 2, w.theta, n, 1, sl7.OUT_STATS, sl7.make_opts(**kw), stats=st)
            ctx.simulate_host_async(w.y0, w.dt, 4, w.theta, n, 1, sl7.OUT_TERMINAL,
                                    sl7.make_opts(prec=sl7.PREC_BF16, colloc=sl7.COLLOC_ANN, **kw),
                                    h_out=np.empty(n, dtype=np.float32))
            ctx.sync()
            torch.cuda.synchronize()
        del st
        torch.cuda.empty_cache()

    cycle()                                   # first use: lazy module / kernel loading
    torch.cuda.synchronize()
    free0, _ = torch.cuda.mem_get_info()
    for _ in range(20):
        cycle()
    torch.cuda.synchronize()
    free1, _ = torch.cuda.mem_get_info()
    assert free0 - free1 < 64 << 20, (free0, free1)


def test_experiment_hook_is_ignored_by_product_builds(gpu_lib, monkeypatch):
    """SL7_TC_VARIANT (the epilogue A/B hook; variant 9 skips the MMAs) is honoured only by -DSL7_AB_HOOKS
    experiment builds: the product library gives bitwise the same results with it set."""
    sl7 = gpu_lib
    torch = _torch()
    w = workloads()["cfg1"]
    ctx = sl7.Context(w.m, list(w.dims), w.act)
    ctx.load_weights(load_golden_blob(w.blob))
    opts = sl7.make_opts(prec=sl7.PREC_BF16, colloc=sl7.COLLOC_ANN)
    ref, _ = ctx.simulate(w.y0, 1 / 8, 8, (), 20_000, 3, sl7.OUT_TERMINAL, opts)
    torch.cuda.synchronize()
    for v in ("1", "9", "11"):
        monkeypatch.setenv("SL7_TC_VARIANT", v)
        out, _ = ctx.simulate(w.y0, 1 / 8, 8, (), 20_000, 3, sl7.OUT_TERMINAL, opts)
        torch.cuda.synchronize()
        assert torch.equal(out, ref), v
