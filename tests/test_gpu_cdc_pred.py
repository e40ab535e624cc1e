"""GPU parity of the 7L-CDC scheme with predicted marginal points (SL7_SCHEME_CDC_PRED, reading R-26 of
DESIGN.md) against the float64 oracle, teacher-forced: per step the oracle recomputes the marginal
points from the predictor at (Y0, t_i), the table and the per-path step from the device's stored states
and the same normals; tolerance 1e-5 * kappa with the CDC forward-error scale.  The scheme couples no
paths, so shards (path_offset) must reproduce the one-call run bit for bit.  m = 5 and 7 run the fused
all-steps kernel, other m the per-step launches."""
import numpy as np
import pytest

from oracle import sl7_oracle as O
from sl7_inputs import load_golden_blob, workloads

pytestmark = pytest.mark.gpu

CASES = [
    ("ou_exact", 7, "ou", (0.0, 1.0, 0.5), 1.0, 0.125, 16),
    ("gbm_exact", 5, "gbm", (0.05, 0.2), 1.0, 0.25, 4),
    ("ou_exact_m6_per_step", 6, "ou", (0.3, 0.7, 0.9), 0.5, 0.25, 7),   # m = 6: the per-step launch path
    ("cfg2_ou_ann", 7, "ann", None, None, None, 16),
    ("cfg0_ann", 5, "ann", None, None, None, 2),
    ("cfg2_cir_ann", 7, "ann", None, None, None, 16),
]


def _setup(sl7, name, m, colloc, theta, y0, dt, n_steps):
    W = workloads()
    if colloc == "ann":
        w = W[{"cfg2_ou_ann": "cfg2_ou", "cfg0_ann": "cfg0", "cfg2_cir_ann": "cfg2_cir"}[name]]
        blob = load_golden_blob(w.blob)
        ctx = sl7.Context(w.m, list(w.dims), w.act)
        ctx.load_weights(blob)
        th = tuple(w.theta) if w.process != "gbm" else ()
        return ctx, sl7.COLLOC_ANN, th, O.Spec(w.m, "ann", th, w.y0, w.dt, n_steps, net=O.parse_blob(blob))
    ctx = sl7.Context(m)
    code = sl7.COLLOC_EXACT_OU if colloc == "ou" else sl7.COLLOC_EXACT_GBM
    return ctx, code, theta, O.Spec(m, colloc, theta, y0, dt, n_steps)


@pytest.mark.parametrize("fast", [False, True])
@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_cdc_pred_teacher_forced(gpu_lib, case, fast):
    import torch
    sl7 = gpu_lib
    name, m, colloc, theta, y0, dt, n_steps = case
    ctx, code, th, spec = _setup(sl7, name, m, colloc, theta, y0, dt, n_steps)
    n_paths = 20_011
    flags = sl7.FLAG_FAST_NORMALS if fast else 0
    opts = sl7.make_opts(prec=sl7.PREC_FP32, colloc=code, scheme=sl7.SCHEME_CDC_PRED, flags=flags)
    out, _ = ctx.simulate(spec.y0, spec.dt, n_steps, th, n_paths, 9, sl7.OUT_FULL, opts)
    torch.cuda.synchronize()
    Yd = out.double().cpu().numpy().reshape(n_steps + 1, n_paths)
    assert np.all(Yd[0] == np.float32(spec.y0))
    assert np.all(np.isfinite(Yd))
    if fast:   # the fast Box-Muller is its own approximation: drive the oracle with the device's normals
        z = torch.empty(n_steps * n_paths, dtype=torch.float32, device="cuda")
        sl7.normals(9, 0, n_paths, n_steps, z, flags=sl7.FLAG_FAST_NORMALS)
        torch.cuda.synchronize()
        Z = z.double().cpu().numpy().reshape(n_steps, n_paths)
    else:
        Z = O.normals(9, np.arange(n_paths, dtype=np.uint64), n_steps)
    worst = 0.0
    with np.errstate(all="ignore"):
        for i in range(n_steps):
            ref = O.cdc_pred_step(spec, i, Yd[i], Z[i])
            kappa = O.cdc_pred_step_error_scale(spec, i, Yd[i], Z[i])
            r = np.abs(Yd[i + 1] - ref) / kappa
            worst = max(worst, float(r.max()))
            assert not (r > 1e-5).any(), "step %d: %d paths off, worst %.3g" % (i, int((r > 1e-5).sum()), r.max())
    print("%s CDC_PRED teacher-forced worst |err|/kappa = %.3g" % (name, worst))


def test_cdc_pred_shards_equal_one_call(gpu_lib):
    # no exchange: two path_offset shards reproduce the one-call FULL output bit for bit
    import torch
    sl7 = gpu_lib
    ctx, code, th, spec = _setup(sl7, "cfg2_cir_ann", 7, "ann", None, None, None, 16)
    n, cut = 50_001, 17_389
    o = sl7.make_opts(colloc=code, scheme=sl7.SCHEME_CDC_PRED)
    full, _ = ctx.simulate(spec.y0, spec.dt, 16, th, n, 3, sl7.OUT_FULL, o)
    a, _ = ctx.simulate(spec.y0, spec.dt, 16, th, cut, 3, sl7.OUT_FULL, o)
    ob = sl7.make_opts(colloc=code, scheme=sl7.SCHEME_CDC_PRED, path_offset=cut)
    b, _ = ctx.simulate(spec.y0, spec.dt, 16, th, n - cut, 3, sl7.OUT_FULL, ob)
    torch.cuda.synchronize()
    F = full.view(17, n).cpu()
    assert torch.equal(F[:, :cut], a.view(17, cut).cpu())
    assert torch.equal(F[:, cut:], b.view(17, n - cut).cpu())


def test_cdc_pred_stats_match_full(gpu_lib):
    import torch
    sl7 = gpu_lib
    ctx, code, th, spec = _setup(sl7, "cfg2_ou_ann", 7, "ann", None, None, None, 16)
    n = 30_000
    o = sl7.make_opts(colloc=code, scheme=sl7.SCHEME_CDC_PRED)
    full, _ = ctx.simulate(spec.y0, spec.dt, 16, th, n, 4, sl7.OUT_FULL, o)
    term, _ = ctx.simulate(spec.y0, spec.dt, 16, th, n, 4, sl7.OUT_TERMINAL, o)
    st = torch.zeros(sl7.stats_elems(64), dtype=torch.float64, device="cuda")
    os_ = sl7.make_opts(colloc=code, scheme=sl7.SCHEME_CDC_PRED, n_bins=64, hist_lo=-3, hist_hi=3, shift=0.0)
    ctx.simulate(spec.y0, spec.dt, 16, th, n, 4, sl7.OUT_STATS, os_, stats=st)
    torch.cuda.synchronize()
    last = full[-n:].double().cpu().numpy()
    assert np.array_equal(last, term.double().cpu().numpy())
    v = O.stats_vector(last, 0.0, -3.0, 3.0, 64)
    s = st.cpu().numpy()
    assert s[0] == n and np.array_equal(s[8:], v[8:])
    np.testing.assert_allclose(s[2:6], v[2:6], rtol=1e-12, atol=1e-9)


@pytest.mark.parametrize("name", ["cfg2_cir", "cfg4", "cfg2_ou"])
def test_cdc_pred_cir_terminal_moments_identical_paths(gpu_lib, name):
    # T-4 on the identical path set: the device's CDC_PRED run of paths 0..2e4-1 against the oracle's
    # free run of the same paths (fp32 table; O3), terminal mean and variance within 1e-4 relative
    import torch
    sl7 = gpu_lib
    w = workloads()[name]
    ctx, code, th, spec = _setup(sl7, "cfg2_ou_ann" if name == "cfg2_ou" else "cfg2_cir_ann", 7, "ann", None, None,
                                 None, w.n_steps)
    spec = O.Spec(w.m, "ann", th, w.y0, w.dt, w.n_steps, net=spec.net)
    n = 20_000
    o = sl7.make_opts(colloc=code, scheme=sl7.SCHEME_CDC_PRED)
    out, _ = ctx.simulate(w.y0, w.dt, w.n_steps, th, n, w.seed, sl7.OUT_TERMINAL, o)
    torch.cuda.synchronize()
    YT = out.double().cpu().numpy()
    with np.errstate(all="ignore"):
        Y, _ = O.simulate_cdc_pred(spec, w.seed, np.arange(n, dtype=np.uint64))
    Yo = Y[-1]
    assert np.all(np.isfinite(YT)) and np.all(np.isfinite(Yo))
    print("%s CDC_PRED: dmean/mean %.2g dvar/var %.2g" % (name, abs(YT.mean() / Yo.mean() - 1),
                                                          abs(YT.var() / Yo.var() - 1)))
    assert abs(YT.mean() - Yo.mean()) <= 1e-4 * abs(Yo.mean())
    assert abs(YT.var() - Yo.var()) <= 1e-4 * Yo.var()
    # the clamp count (stats E1 of a CDC_PRED run) against the oracle's count on the same paths: fp32 and
    # fp64 states can fall on different sides of a hull edge, hence the small allowance
    st = torch.zeros(sl7.stats_elems(0), dtype=torch.float64, device="cuda")
    os_ = sl7.make_opts(colloc=code, scheme=sl7.SCHEME_CDC_PRED, shift=0.1)
    ctx.simulate(w.y0, w.dt, w.n_steps, th, n, w.seed, sl7.OUT_STATS, os_, stats=st)
    torch.cuda.synchronize()
    nd, no = st[6].item(), O.cdc_pred_clamped(spec, Y)
    print("%s CDC_PRED clamped path-steps: device %d oracle %d" % (name, nd, no))
    assert no > 0 and abs(nd - no) <= 0.005 * no + 10
    assert sl7.stats_summary(st.cpu().numpy(), os_)["clamped_steps"] == nd


@pytest.mark.parametrize("name", ["cfg2_cir", "cfg4"])
def test_cdc_pred_cir_full_size_law(gpu_lib, name):
    # cfg2 (1e8 paths, T = 2) and cfg4's shape (1e8 paths, T = 4): every path finite (the empirical-quantile
    # CDC diverges here, R-25) and the terminal mean within 1% of the CIR law
    # E Y_T = Y0 e^{-kT} + Ybar (1 - e^{-kT}) -- the network is fitted for horizons up to 4 (R-26)
    import torch
    sl7 = gpu_lib
    w = workloads()[name]
    ctx, code, th, _ = _setup(sl7, "cfg2_cir_ann", 7, "ann", None, None, None, w.n_steps)
    st = torch.zeros(sl7.stats_elems(4096), dtype=torch.float64, device="cuda")
    o = sl7.make_opts(colloc=code, scheme=sl7.SCHEME_CDC_PRED, n_bins=4096, hist_lo=0.0, hist_hi=0.8, shift=0.1)
    ctx.simulate(w.y0, w.dt, w.n_steps, th, 100_000_000, w.seed, sl7.OUT_STATS, o, stats=st)
    torch.cuda.synchronize()
    v = st.cpu().numpy()
    assert v[0] == 100_000_000 and v[1] == 0                     # count, non-finite count
    k, yb, _ = w.theta
    e = np.exp(-k * w.T)
    law = w.y0 * e + yb * (1 - e)
    mean = 0.1 + v[2] / v[0]
    print("%s CDC_PRED mean %.6f law %.6f" % (name, mean, law))
    assert abs(mean / law - 1) < 0.01


def test_cdc_pred_refuses_horizons_outside_the_fit(gpu_lib):
    # the blob's fitted box (flags bit 2): dt 0.5 x 16 steps reads the predictor at t = 7.5 > 4
    sl7 = gpu_lib
    w = workloads()["cfg2_cir"]
    ctx, code, th, _ = _setup(sl7, "cfg2_cir_ann", 7, "ann", None, None, None, w.n_steps)
    o = sl7.make_opts(colloc=code, scheme=sl7.SCHEME_CDC_PRED)
    with pytest.raises(sl7.Sl7Error, match="fitted dt range"):
        ctx.simulate(w.y0, 0.5, 16, th, 1024, w.seed, sl7.OUT_TERMINAL, o)


@pytest.mark.parametrize("mode", ["full", "terminal"])
def test_cdc_pred_fused_edge_sizes(gpu_lib, mode):
    # ragged path counts around the fused kernel's 1024-path groups and step counts not a multiple of 4:
    # terminal values equal the oracle's free-running paths within the fp32 tolerance
    import torch
    sl7 = gpu_lib
    ctx = sl7.Context(5)
    th = (0.4, 0.8, 0.6)
    for n_paths, n_steps in [(1, 1), (1023, 3), (1025, 5), (4097, 9)]:
        o = sl7.make_opts(colloc=sl7.COLLOC_EXACT_OU, scheme=sl7.SCHEME_CDC_PRED)
        out_mode = sl7.OUT_FULL if mode == "full" else sl7.OUT_TERMINAL
        out, _ = ctx.simulate(0.7, 0.2, n_steps, th, n_paths, 21, out_mode, o)
        torch.cuda.synchronize()
        spec = O.Spec(5, "ou", th, 0.7, 0.2, n_steps)
        Y, _ = O.simulate_cdc_pred(spec, 21, np.arange(n_paths, dtype=np.uint64))
        got = out.double().cpu().numpy().reshape(-1, n_paths)
        ref = Y if mode == "full" else Y[-1:]
        np.testing.assert_allclose(got, ref, rtol=2e-5, atol=2e-5)


@pytest.mark.parametrize("entry", ["host", "host_async"])
def test_cdc_pred_host_entry_points_equal_simulate(gpu_lib, entry):
    # sl7_simulate_host / _async build the per-step predictor horizons themselves: on a fresh
    # context, and after an earlier call with other (Y0, dt, n_steps) -- stale horizons would change the paths
    import torch
    sl7 = gpu_lib
    ctx, code, th, spec = _setup(sl7, "cfg2_ou_ann", 7, "ann", None, None, None, 16)
    n = 5_003
    o = sl7.make_opts(colloc=code, scheme=sl7.SCHEME_CDC_PRED)
    ref_ctx, _, _, _ = _setup(sl7, "cfg2_ou_ann", 7, "ann", None, None, None, 16)
    ref, _ = ref_ctx.simulate(spec.y0, spec.dt, 16, th, n, 5, sl7.OUT_FULL, o)
    ref_short, _ = ref_ctx.simulate(0.4, 0.05, 6, th, n, 5, sl7.OUT_FULL, o)
    torch.cuda.synchronize()
    for y0, dt, ns, want in ((spec.y0, spec.dt, 16, ref), (0.4, 0.05, 6, ref_short), (spec.y0, spec.dt, 16, ref)):
        h = np.empty(sl7.out_elems(ns, n, sl7.OUT_FULL), dtype=np.float32)
        if entry == "host":
            ctx.simulate_host(y0, dt, ns, th, n, 5, sl7.OUT_FULL, o, h_out=h)
        else:
            ctx.simulate_host_async(y0, dt, ns, th, n, 5, sl7.OUT_FULL, o, h_out=h)
            ctx.sync()
        assert np.array_equal(h, want.cpu().numpy())


@pytest.mark.parametrize("case", [CASES[0], CASES[2]], ids=["fused_m7", "per_step_m6"])
def test_cdc_pred_clamp_count_both_launch_paths(gpu_lib, case):
    # stats E1 of CDC_PRED = clamped path-steps, from the fused kernel (m = 7) and from the per-step launches
    # (m = 6, counts added into the stats vector after every step) against the oracle's count
    import torch
    sl7 = gpu_lib
    name, m, colloc, theta, y0, dt, n_steps = case
    ctx, code, th, spec = _setup(sl7, name, m, colloc, theta, y0, dt, n_steps)
    n = 20_000
    out, _ = ctx.simulate(spec.y0, spec.dt, n_steps, th, n, 13, sl7.OUT_FULL,
                          sl7.make_opts(colloc=code, scheme=sl7.SCHEME_CDC_PRED))
    st = torch.zeros(sl7.stats_elems(0), dtype=torch.float64, device="cuda")
    ctx.simulate(spec.y0, spec.dt, n_steps, th, n, 13, sl7.OUT_STATS,
                 sl7.make_opts(colloc=code, scheme=sl7.SCHEME_CDC_PRED, shift=spec.y0), stats=st)
    torch.cuda.synchronize()
    Yd = out.double().cpu().numpy().reshape(n_steps + 1, n)
    nd, no = st[6].item(), O.cdc_pred_clamped(spec, Yd)   # the oracle counts on the device's own states
    print("%s clamped path-steps: device %d oracle %d" % (name, nd, no))
    assert no > 0 and abs(nd - no) <= 2
