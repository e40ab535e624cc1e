"""GPU parity of the 7L-CDC scheme (SL7_SCHEME_CDC) against the float64 oracle, teacher-forced:
for every step the oracle recomputes the marginal points, the table and the per-path step from the
device's own states of ALL paths (FULL output) and the same normals; tolerance 1e-5 * kappa with the
CDC forward-error scale (oracle.cdc_step_error_scale)."""
import numpy as np
import pytest

from oracle import sl7_oracle as O
from sl7_inputs import load_golden_blob, workloads

pytestmark = pytest.mark.gpu

CASES = [
    ("ou_exact", 7, "ou", (0.0, 1.0, 0.5), 1.0, 0.125, 16),
    ("gbm_exact", 5, "gbm", (0.05, 0.2), 1.0, 0.25, 4),
    ("cfg2_ou_ann", 7, "ann", None, None, None, 6),
    ("cfg0_ann", 5, "ann", None, None, None, 2),
    ("cfg2_cir_ann", 7, "ann", None, None, None, 5),
]


def _setup(sl7, name, m, colloc, theta, y0, dt, n_steps):
    W = workloads()
    if colloc == "ann":
        w = W[{"cfg2_ou_ann": "cfg2_ou", "cfg0_ann": "cfg0", "cfg2_cir_ann": "cfg2_cir"}[name]]
        blob = load_golden_blob(w.blob)
        ctx = sl7.Context(w.m, list(w.dims), w.act)
        ctx.load_weights(blob)
        th = tuple(w.theta) if w.process != "gbm" else ()
        spec = O.Spec(w.m, "ann", th, w.y0, w.dt, n_steps, net=O.parse_blob(blob))
        return ctx, sl7.COLLOC_ANN, th, spec
    ctx = sl7.Context(m)
    code = sl7.COLLOC_EXACT_OU if colloc == "ou" else sl7.COLLOC_EXACT_GBM
    return ctx, code, theta, O.Spec(m, colloc, theta, y0, dt, n_steps)


@pytest.mark.parametrize("fast", [False, True])
@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_cdc_teacher_forced(gpu_lib, case, fast):
    import torch
    sl7 = gpu_lib
    name, m, colloc, theta, y0, dt, n_steps = case
    ctx, code, th, spec = _setup(sl7, name, m, colloc, theta, y0, dt, n_steps)
    n_paths = 20_011
    flags = sl7.FLAG_FAST_NORMALS if fast else 0
    opts = sl7.make_opts(prec=sl7.PREC_FP32, colloc=code, scheme=sl7.SCHEME_CDC, flags=flags)
    out, _ = ctx.simulate(spec.y0, spec.dt, n_steps, th, n_paths, 9, sl7.OUT_FULL, opts)
    torch.cuda.synchronize()
    Yd = out.double().cpu().numpy().reshape(n_steps + 1, n_paths)
    assert np.all(Yd[0] == np.float32(spec.y0))
    if fast:   # the fast Box-Muller is its own approximation: drive the oracle with the device's normals
        z = torch.empty(n_steps * n_paths, dtype=torch.float32, device="cuda")
        sl7.normals(9, 0, n_paths, n_steps, z, flags=sl7.FLAG_FAST_NORMALS)
        torch.cuda.synchronize()
        Z = z.double().cpu().numpy().reshape(n_steps, n_paths)
    else:
        Z = O.normals(9, np.arange(n_paths, dtype=np.uint64), n_steps)
    worst = 0.0
    for i in range(n_steps):
        ref = O.cdc_step(spec, Yd[i], Z[i])
        kappa = O.cdc_step_error_scale(spec, Yd[i], Z[i])
        r = np.abs(Yd[i + 1] - ref) / kappa
        worst = max(worst, float(r.max()))
        assert not (r > 1e-5).any(), "step %d: %d paths off, worst %.3g" % (i, int((r > 1e-5).sum()), r.max())
    print("%s CDC teacher-forced worst |err|/kappa = %.3g" % (name, worst))


def test_cdc_terminal_and_stats_match_full(gpu_lib):
    import torch
    sl7 = gpu_lib
    ctx, code, th, spec = _setup(sl7, "ou_exact", 7, "ou", (0.0, 1.0, 0.5), 1.0, 0.125, 9)
    n = 30_000
    o = sl7.make_opts(colloc=code, scheme=sl7.SCHEME_CDC)
    full, _ = ctx.simulate(1.0, 0.125, 9, th, n, 4, sl7.OUT_FULL, o)
    term, _ = ctx.simulate(1.0, 0.125, 9, th, n, 4, sl7.OUT_TERMINAL, o)
    st = torch.zeros(sl7.stats_elems(64), dtype=torch.float64, device="cuda")
    os_ = sl7.make_opts(colloc=code, scheme=sl7.SCHEME_CDC, n_bins=64, hist_lo=-3, hist_hi=3, shift=0.0)
    ctx.simulate(1.0, 0.125, 9, th, n, 4, sl7.OUT_STATS, os_, stats=st)
    torch.cuda.synchronize()
    last = full[-n:].double().cpu().numpy()
    assert np.array_equal(last, term.double().cpu().numpy())
    v = O.stats_vector(last, 0.0, -3.0, 3.0, 64)
    s = st.cpu().numpy()
    assert s[0] == n and np.array_equal(s[8:], v[8:])
    np.testing.assert_allclose(s[2:6], v[2:6], rtol=1e-12, atol=1e-9)


def test_cdc_rejects_reference_and_tc(gpu_lib):
    sl7 = gpu_lib
    ctx = sl7.Context(5)
    o = sl7.make_opts(colloc=sl7.COLLOC_EXACT_GBM, scheme=sl7.SCHEME_CDC, ref=sl7.REF_GBM, ref_theta=(0.05, 0.2, 0))
    with pytest.raises(sl7.Sl7Error, match="EUNSUPPORTED"):
        ctx.simulate(1.0, 0.5, 2, (0.05, 0.2), 100, 1, sl7.OUT_TERMINAL, o)


@pytest.mark.parametrize("name", ["ou_exact", "cfg2_ou_ann"])
def test_cdc_terminal_moments_identical_paths(gpu_lib, name):
    """T-4 for the quantile-marginal 7L-CDC: the device runs the 2e4 paths of one call free from Y0 (their own
    empirical quantiles each step), the oracle runs the same path set with its float64 quantiles; terminal mean
    and variance within 1e-4 relative (cfg2's OU network over its 16 steps, and exact OU collocation)."""
    import torch
    sl7 = gpu_lib
    case = {c[0]: c for c in CASES}[name]
    _, m, colloc, theta, y0, dt, _ = case
    ctx, code, th, spec = _setup(sl7, name, m, colloc, theta, y0, dt, 16)
    n = 20_000
    opts = sl7.make_opts(prec=sl7.PREC_FP32, colloc=code, scheme=sl7.SCHEME_CDC)
    out, _ = ctx.simulate(spec.y0, spec.dt, 16, th, n, 11, sl7.OUT_TERMINAL, opts)
    torch.cuda.synchronize()
    YT = out.double().cpu().numpy()
    with np.errstate(all="ignore"):
        Y, _ = O.simulate_cdc(spec, 11, np.arange(n, dtype=np.uint64))
    Yo = Y[-1]
    assert np.all(np.isfinite(YT)) and np.all(np.isfinite(Yo))
    mo, vo = Yo.mean(), Yo.var()
    scale = abs(mo) if abs(mo) >= 1e-3 * np.sqrt(vo) else np.sqrt(vo)
    print("%s CDC: dmean/scale %.2g dvar/var %.2g" % (name, abs(YT.mean() - mo) / scale, abs(YT.var() - vo) / vo))
    assert abs(YT.mean() - mo) <= 1e-4 * scale
    assert abs(YT.var() - vo) <= 1e-4 * vo
