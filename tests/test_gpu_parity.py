"""GPU parity: the CUDA path (through the C ABI) against the float64 oracle, element by element.

Tolerances (BASELINE north_star):
  T-1 Philox words bit-exact (and equal to cuRAND curand4());
  T-2 fp32 path values: teacher-forced one step, |Y_dev - Y_or| <= 1e-5 * kappa, kappa the
      forward-error scale sum_j |l_j(Z)| A_j;
  T-5 histogram counts equal except values within one fp32 ulp of an edge;
  T-6 sharded runs bitwise equal per path, histogram equal, moments within 1e-12.
"""
import ctypes
import os

import numpy as np
import pytest

from oracle import sl7_oracle as O
from sl7_inputs import ACT_SOFTPLUS, ACT_TANH, glorot_mlp, load_golden_blob, pack_blob, workloads

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _torch():
    import torch
    return torch


def _run(sl7, ctx, spec_kw, n_paths, seed, out_mode=None, colloc=None, prec=None, stats=False, n_bins=0,
         lo=0.0, hi=1.0, shift=0.0, ref=0, ref_theta=(0, 0, 0), offset=0, theta=None, flags=0):
    torch = _torch()
    opts = sl7.make_opts(prec=sl7.PREC_FP32 if prec is None else prec, colloc=colloc, path_offset=offset,
                         n_bins=n_bins, hist_lo=lo, hist_hi=hi, shift=shift, ref=ref, ref_theta=ref_theta,
                         flags=flags)
    st = torch.zeros(sl7.stats_elems(n_bins), dtype=torch.float64, device="cuda") if stats else None
    out, st = ctx.simulate(spec_kw["y0"], spec_kw["dt"], spec_kw["n_steps"], theta, n_paths, seed, out_mode, opts,
                           stats=st)
    torch.cuda.synchronize()
    o = None if out is None else out.double().cpu().numpy()
    return o, (None if st is None else st.cpu().numpy())


def _teacher_forced(spec, Yd, Z, tol=1e-5):
    worst = 0.0
    for i in range(spec.n_steps):
        ref = O.step(spec, Yd[i], Z[i])
        kappa = O.step_error_scale(spec, Yd[i], Z[i])
        r = np.abs(Yd[i + 1] - ref) / kappa
        worst = max(worst, float(r.max()))
        bad = r > tol
        assert not bad.any(), "step %d: %d/%d paths off, worst %.3g (path %d: dev %r or %r)" % (
            i, bad.sum(), bad.size, r.max(), int(np.argmax(r)), Yd[i + 1][np.argmax(r)], ref[np.argmax(r)])
    return worst


# ------------------------------------------------------------------------------------------- RNG

@pytest.mark.parametrize("offset", [0, (1 << 32) - 300, (1 << 64) - 1000])
def test_philox_bitexact_vs_oracle(gpu_lib, offset):
    torch = _torch()
    sl7 = gpu_lib
    n = 1000 if offset else 70_001
    for seed, block in [(2302051701, 0), (0xFFFFFFFFFFFFFFFF, 7), (123, 0xFFFFFFFF)]:
        out = torch.empty(4 * n, dtype=torch.int32, device="cuda")
        sl7.philox_u32(seed, offset, n, block, out)
        torch.cuda.synchronize()
        dev = out.cpu().numpy().view(np.uint32).reshape(4, n)
        ref = O.philox_block(seed, np.uint64(offset) + np.arange(n, dtype=np.uint64), block)
        for k in range(4):
            np.testing.assert_array_equal(dev[k], ref[k].astype(np.uint32))


def test_philox_equals_curand(gpu_lib):
    torch = _torch()
    sl7 = gpu_lib
    lib = ctypes.CDLL(os.path.join(ROOT, "tests", "native", "libcurand_pin.so"))
    lib.curand_pin_u32.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint32,
                                   ctypes.c_void_p, ctypes.c_void_p]
    n = 50_000
    for seed, off, block in [(2302051701, 0, 0), (99, (1 << 33) + 5, 3), (0xDEADBEEFCAFEF00D, 17, 1000)]:
        a = torch.empty(4 * n, dtype=torch.int32, device="cuda")
        b = torch.empty(4 * n, dtype=torch.int32, device="cuda")
        sl7.philox_u32(seed, off, n, block, a)
        assert lib.curand_pin_u32(seed, off, n, block, ctypes.c_void_p(b.data_ptr()),
                                  ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)) == 0
        torch.cuda.synchronize()
        assert torch.equal(a, b)


def test_normals_vs_oracle(gpu_lib):
    torch = _torch()
    sl7 = gpu_lib
    n, steps, seed = 200_000, 9, 77
    out = torch.empty(steps * n, dtype=torch.float32, device="cuda")
    sl7.normals(seed, 5, n, steps, out)
    torch.cuda.synchronize()
    dev = out.double().cpu().numpy().reshape(steps, n)
    ref = O.normals(seed, 5 + np.arange(n, dtype=np.uint64), steps)
    err = np.abs(dev - ref)
    assert err.max() <= 2e-6 * np.maximum(1.0, np.abs(ref)).max()
    assert np.all(err <= 1e-6 * np.maximum(1.0, np.abs(ref)))


# ----------------------------------------------------------------------------------- exact modes

@pytest.mark.parametrize("m,n_steps,dt", [(5, 2, 0.5), (7, 64, 1 / 64), (3, 5, 0.3), (1, 3, 0.5), (12, 4, 1.0)])
def test_exact_gbm_full_teacher_forced(gpu_lib, m, n_steps, dt):
    sl7 = gpu_lib
    n_paths = 20_000 + 33
    ctx = sl7.Context(m)
    kw = dict(y0=1.0, dt=dt, n_steps=n_steps)
    Yd, _ = _run(sl7, ctx, kw, n_paths, 2302051700, sl7.OUT_FULL, sl7.COLLOC_EXACT_GBM, theta=(0.05, 0.2))
    Yd = Yd.reshape(n_steps + 1, n_paths)
    assert np.all(Yd[0] == 1.0)
    spec = O.Spec(m, "gbm", (0.05, 0.2), 1.0, dt, n_steps)
    Z = O.normals(2302051700, np.arange(n_paths, dtype=np.uint64), n_steps)
    _teacher_forced(spec, Yd, Z)
    # free running: drift of fp32 vs fp64 stays small (reported bound)
    Yo, _ = O.simulate(spec, 2302051700, np.arange(n_paths, dtype=np.uint64))
    rel = np.abs(Yd[-1] - Yo[-1]) / np.abs(Yo[-1])
    assert np.median(rel) < 1e-5 and rel.max() < 5e-4


@pytest.mark.parametrize("theta", [(0.0, 1.0, 0.5), (0.3, 1e-8, 0.7), (-0.2, 3.0, 0.0)])
def test_exact_ou_full_teacher_forced_and_eq66(gpu_lib, theta):
    sl7 = gpu_lib
    n_paths, n_steps, dt = 30_000, 16, 0.125
    ctx = sl7.Context(7)
    Yd, _ = _run(sl7, ctx, dict(y0=1.0, dt=dt, n_steps=n_steps), n_paths, 5, sl7.OUT_FULL, sl7.COLLOC_EXACT_OU,
                 theta=theta)
    Yd = Yd.reshape(n_steps + 1, n_paths)
    spec = O.Spec(7, "ou", theta, 1.0, dt, n_steps)
    Z = O.normals(5, np.arange(n_paths, dtype=np.uint64), n_steps)
    _teacher_forced(spec, Yd, Z)
    R = O.exact_reference("ou", theta, 1.0, dt, Z)           # Eq. 6.6 on the same normals
    assert np.max(np.abs(Yd[-1] - R)) < 2e-5


def test_sigma_zero_and_degenerate_sizes(gpu_lib):
    sl7 = gpu_lib
    ctx = sl7.Context(5)
    Yd, _ = _run(sl7, ctx, dict(y0=2.0, dt=0.25, n_steps=4), 1, 9, sl7.OUT_FULL, sl7.COLLOC_EXACT_GBM,
                 theta=(0.05, 0.0))
    np.testing.assert_allclose(Yd, 2.0 * np.exp(0.05 * 0.25 * np.arange(5)), rtol=3e-7)
    Yd, _ = _run(sl7, ctx, dict(y0=1.0, dt=0.5, n_steps=1), 257, 9, sl7.OUT_TERMINAL, sl7.COLLOC_EXACT_OU,
                 theta=(0.1, 1.0, 0.0))
    np.testing.assert_allclose(Yd, np.exp(-0.5) + 0.1 * (1 - np.exp(-0.5)), rtol=3e-7)


# ------------------------------------------------------------------------------------ ANN-FP32

ANN_CASES = [
    ("cfg0", None),
    ("cfg1", None),
    ("cfg2_ou", None),
    ("cfg2_cir", None),
    ("glorot_generic", ((4, 17, 9, 33, 6), ACT_TANH)),
    ("glorot_generic_sp", ((3, 64, 64, 3), ACT_SOFTPLUS)),
    ("glorot_max_shape", ((2, 64, 64, 64, 64, 64, 64, 16), ACT_TANH)),   # 6 hidden layers, width 64, m = 16
    ("glorot_w50_abs", ((2, 50, 50, 50, 7), ACT_TANH)),                  # golden shape, absolute output form
    ("glorot_w50_res", ((5, 50, 50, 50, 50, 7), ACT_SOFTPLUS, "residual")),
    ("glorot_w64_res", ((3, 64, 64, 5), ACT_TANH, "residual")),
]


def _ann_case(name, gen):
    W = workloads()
    if gen is None:
        w = W[name]
        blob = load_golden_blob(w.blob)
        theta = tuple(w.theta) if w.process != "gbm" else ()
        return blob, w.m, list(w.dims), w.act, theta, w.y0, min(w.n_steps, 16), w.dt
    dims, act = gen[:2]
    p = glorot_mlp(dims, act, seed=31, with_norm=True, residual=len(gen) > 2)
    theta = tuple(0.1 * (k + 1) for k in range(dims[0] - 2))
    return pack_blob(p), dims[-1], list(dims), act, theta, 0.7, 6, 0.2


@pytest.mark.parametrize("name,gen", ANN_CASES, ids=[c[0] for c in ANN_CASES])
def test_ann_fp32_full_teacher_forced(gpu_lib, name, gen):
    sl7 = gpu_lib
    blob, m, dims, act, theta, y0, n_steps, dt = _ann_case(name, gen)
    n_paths = 8192 + 129
    ctx = sl7.Context(m, dims, act)
    ctx.load_weights(blob)
    Yd, _ = _run(sl7, ctx, dict(y0=y0, dt=dt, n_steps=n_steps), n_paths, 424242, sl7.OUT_FULL, sl7.COLLOC_ANN,
                 theta=theta)
    Yd = Yd.reshape(n_steps + 1, n_paths)
    spec = O.Spec(m, "ann", theta, y0, dt, n_steps, net=O.parse_blob(blob))
    Z = O.normals(424242, np.arange(n_paths, dtype=np.uint64), n_steps)
    _teacher_forced(spec, Yd, Z)


def test_ann_requires_weights_and_supported_precision(gpu_lib):
    sl7 = gpu_lib
    w = workloads()["cfg0"]
    ctx = sl7.Context(w.m, list(w.dims), w.act)
    with pytest.raises(sl7.Sl7Error, match="ESTATE"):
        _run(sl7, ctx, dict(y0=1.0, dt=0.5, n_steps=2), 100, 1, sl7.OUT_TERMINAL, sl7.COLLOC_ANN, theta=())
    bad = bytearray(load_golden_blob(w.blob))
    bad[4] = 9
    with pytest.raises(sl7.Sl7Error, match="version"):
        ctx.load_weights(bytes(bad))
    with pytest.raises(sl7.Sl7Error, match="EFORMAT"):
        ctx.load_weights(load_golden_blob(w.blob)[:-4])
    bad = bytearray(load_golden_blob(w.blob))
    fo = 12 + 4 * len(w.dims) + 4                      # flags word (include/sl7.h 'Weights blob')
    bad[fo] |= 8                                       # unknown flag bit (bits 0-2 are defined)
    with pytest.raises(sl7.Sl7Error, match="flags"):
        ctx.load_weights(bytes(bad))


# ------------------------------------------------------------------------------------ statistics

def test_stats_fused_vs_oracle(gpu_lib):
    sl7 = gpu_lib
    n_paths, n_bins, lo, hi = 300_007, 4096, 0.0, 3.0
    ctx = sl7.Context(7)
    kw = dict(y0=1.0, dt=1 / 16, n_steps=16)
    YT, st = _run(sl7, ctx, kw, n_paths, 11, sl7.OUT_TERMINAL, sl7.COLLOC_EXACT_GBM, stats=True, n_bins=n_bins,
                  lo=lo, hi=hi, shift=1.0, ref=sl7.REF_GBM, ref_theta=(0.05, 0.2, 0), theta=(0.05, 0.2))
    # the reference Y(T) is evaluated on the normals the kernel consumed (fp32 X_hat, the same inputs):
    # the exact-mode strong error is rounding-level (~3e-7), the size of the fp32-vs-fp64 normal gap
    torch = _torch()
    zd = torch.empty(16 * n_paths, dtype=torch.float32, device="cuda")
    sl7.normals(11, 0, n_paths, 16, zd)
    torch.cuda.synchronize()
    Zd = zd.double().cpu().numpy().reshape(16, n_paths)
    R = O.exact_reference("gbm", (0.05, 0.2), 1.0, 1 / 16, Zd)
    v = O.stats_vector(YT, 1.0, lo, hi, n_bins, R)            # same terminal values, oracle statistics
    assert st[0] == v[0] and st[1] == 0
    np.testing.assert_allclose(st[2:6], v[2:6], rtol=1e-12, atol=1e-9)
    np.testing.assert_allclose(st[6:8], v[6:8], rtol=1e-7)
    w = (hi - lo) / n_bins
    edge = np.abs((YT - lo) / w - np.round((YT - lo) / w)) * w <= np.spacing(YT.astype(np.float32)).astype(np.float64)
    diff = np.abs(st[8:] - v[8:]).sum()
    assert diff <= 2 * edge.sum()
    # strong error of exact GBM collocation vs exact GBM: rounding-level, flat in dt
    assert st[6] / st[0] < 5e-6


def test_sharding_bitwise(gpu_lib):
    """T-6: per-path outputs of W shards (path_offset) are bitwise the unsharded run's."""
    sl7 = gpu_lib
    torch = _torch()
    w = workloads()["cfg2_ou"]
    blob = load_golden_blob(w.blob)
    ctx = sl7.Context(w.m, list(w.dims), w.act)
    ctx.load_weights(blob)
    N = 100_003
    kw = dict(y0=w.y0, dt=w.dt, n_steps=w.n_steps)
    full, st_full = _run(sl7, ctx, kw, N, w.seed, sl7.OUT_TERMINAL, sl7.COLLOC_ANN, stats=True, n_bins=512, lo=-2,
                         hi=2, theta=w.theta)
    for W in (2, 3, 8):
        per = -(-N // W)
        parts, acc = [], np.zeros_like(st_full)
        for r in range(W):
            lo_, n = r * per, min(N, (r + 1) * per) - r * per
            o, s = _run(sl7, ctx, kw, n, w.seed, sl7.OUT_TERMINAL, sl7.COLLOC_ANN, stats=True, n_bins=512, lo=-2,
                        hi=2, offset=lo_, theta=w.theta)
            parts.append(o)
            acc += s
        assert np.array_equal(np.concatenate(parts), full)
        assert np.array_equal(acc[8:], st_full[8:]) and acc[0] == st_full[0]
        np.testing.assert_allclose(acc[2:6], st_full[2:6], rtol=1e-12)


def test_host_buffers_equal_device_run(gpu_lib):
    sl7 = gpu_lib
    w = workloads()["cfg0"]
    blob = load_golden_blob(w.blob)
    ctx = sl7.Context(w.m, list(w.dims), w.act)
    ctx.load_weights(blob)
    n = 12_345
    dev, dst = _run(sl7, ctx, dict(y0=1.0, dt=0.5, n_steps=2), n, 3, sl7.OUT_FULL, sl7.COLLOC_ANN, stats=True,
                    n_bins=64, lo=0, hi=3, theta=())
    h_out = np.empty(3 * n, dtype=np.float32)
    h_st = np.empty(sl7.stats_elems(64), dtype=np.float64)
    opts = sl7.make_opts(prec=sl7.PREC_FP32, colloc=sl7.COLLOC_ANN, n_bins=64, hist_lo=0, hist_hi=3)
    _, _, up, down = ctx.simulate_host(1.0, 0.5, 2, (), n, 3, sl7.OUT_FULL, opts, h_out, h_st)
    assert np.array_equal(h_out.astype(np.float64), dev)
    np.testing.assert_allclose(h_st, dst, rtol=1e-12)
    assert down == h_out.nbytes + h_st.nbytes and up > 0


# ------------------------------------------------------------------------------ ANN-BF16 (tcgen05)

@pytest.mark.parametrize("name,gen", ANN_CASES, ids=[c[0] for c in ANN_CASES])
def test_ann_bf16_tc_teacher_forced(gpu_lib, name, gen):
    """T-3: tensor-core path within 5e-3 * kappa of the quantisation-aware oracle O6, one step at a time."""
    sl7 = gpu_lib
    blob, m, dims, act, theta, y0, n_steps, dt = _ann_case(name, gen)
    n_paths = 4 * 128 * 3 + 77                       # several tiles per group, a ragged last tile
    ctx = sl7.Context(m, dims, act)
    ctx.load_weights(blob)
    Yd, _ = _run(sl7, ctx, dict(y0=y0, dt=dt, n_steps=n_steps), n_paths, 99, sl7.OUT_FULL, sl7.COLLOC_ANN,
                 prec=sl7.PREC_BF16, theta=theta)
    Yd = Yd.reshape(n_steps + 1, n_paths)
    spec = O.Spec(m, "ann", theta, y0, dt, n_steps, net=O.parse_blob(blob), quant="bf16")
    Z = O.normals(99, np.arange(n_paths, dtype=np.uint64), n_steps)
    worst = _teacher_forced(spec, Yd, Z, tol=5e-3)
    print("bf16 teacher-forced worst |err|/kappa = %.3g" % worst)


@pytest.mark.parametrize("name,gen", ANN_CASES, ids=[c[0] for c in ANN_CASES])
def test_ann_tf32_tc_teacher_forced(gpu_lib, name, gen):
    """T-3 for SL7_PREC_TF32 (tcgen05 kind::tf32): within 5e-3 * kappa of O6 with TF32 (cvt.rna) rounding."""
    sl7 = gpu_lib
    blob, m, dims, act, theta, y0, n_steps, dt = _ann_case(name, gen)
    n_paths = 4 * 128 * 3 + 51
    ctx = sl7.Context(m, dims, act)
    ctx.load_weights(blob)
    Yd, _ = _run(sl7, ctx, dict(y0=y0, dt=dt, n_steps=n_steps), n_paths, 57, sl7.OUT_FULL, sl7.COLLOC_ANN,
                 prec=sl7.PREC_TF32, theta=theta)
    Yd = Yd.reshape(n_steps + 1, n_paths)
    spec = O.Spec(m, "ann", theta, y0, dt, n_steps, net=O.parse_blob(blob), quant="tf32")
    Z = O.normals(57, np.arange(n_paths, dtype=np.uint64), n_steps)
    worst = _teacher_forced(spec, Yd, Z, tol=5e-3)
    print("tf32 teacher-forced worst |err|/kappa = %.3g" % worst)


@pytest.mark.parametrize("name,gen", ANN_CASES, ids=[c[0] for c in ANN_CASES])
def test_ann_split_tc_teacher_forced(gpu_lib, name, gen):
    """SL7_PREC_SPLIT: bf16 tensor cores with three-part operands reach the fp32 bar (T-2, 1e-5 kappa)
    against the plain float64 oracle O3."""
    sl7 = gpu_lib
    blob, m, dims, act, theta, y0, n_steps, dt = _ann_case(name, gen)
    n_paths = 3 * 128 * 4 + 33
    ctx = sl7.Context(m, dims, act)
    ctx.load_weights(blob)
    Yd, _ = _run(sl7, ctx, dict(y0=y0, dt=dt, n_steps=n_steps), n_paths, 31, sl7.OUT_FULL, sl7.COLLOC_ANN,
                 prec=sl7.PREC_SPLIT, theta=theta)
    Yd = Yd.reshape(n_steps + 1, n_paths)
    spec = O.Spec(m, "ann", theta, y0, dt, n_steps, net=O.parse_blob(blob))
    Z = O.normals(31, np.arange(n_paths, dtype=np.uint64), n_steps)
    worst = _teacher_forced(spec, Yd, Z, tol=1e-5)
    print("split teacher-forced worst |err|/kappa = %.3g" % worst)


def test_ann_bf16_sharding_bitwise(gpu_lib):
    sl7 = gpu_lib
    w = workloads()["cfg0"]
    blob = load_golden_blob(w.blob)
    ctx = sl7.Context(w.m, list(w.dims), w.act)
    ctx.load_weights(blob)
    N = 3 * 512 + 5
    kw = dict(y0=w.y0, dt=w.dt, n_steps=w.n_steps)
    full, _ = _run(sl7, ctx, kw, N, w.seed, sl7.OUT_TERMINAL, sl7.COLLOC_ANN, prec=sl7.PREC_BF16, theta=())
    parts = []
    for lo, n in [(0, 700), (700, 129), (829, N - 829)]:
        o, _ = _run(sl7, ctx, kw, n, w.seed, sl7.OUT_TERMINAL, sl7.COLLOC_ANN, prec=sl7.PREC_BF16, offset=lo, theta=())
        parts.append(o)
    assert np.array_equal(np.concatenate(parts), full)


# ------------------------------------------------------------- exact modes: fast RNG + closed-form g_m

@pytest.mark.parametrize("colloc,m,theta,n_steps,dt", [
    ("gbm", 5, (0.05, 0.2), 64, 1 / 64), ("gbm", 7, (0.05, 0.2), 4, 1.0), ("gbm", 8, (0.1, 0.5), 6, 0.5),
    ("gbm", 3, (0.05, 0.2), 5, 0.3), ("ou", 7, (0.0, 1.0, 0.5), 16, 0.125), ("ou", 5, (0.3, 1e-9, 0.7), 9, 0.25)])
@pytest.mark.parametrize("flags", [1, 2, 3])
def test_exact_flags_teacher_forced(gpu_lib, colloc, m, theta, n_steps, dt, flags):
    """SL7_FLAG_SPECIALIZED (closed-form g_m) keeps the fp32 tolerance 1e-5 * kappa against the float64
    oracle; under SL7_FLAG_FAST_NORMALS the oracle is driven by the device's fast normals (their own
    accuracy, 2e-6 (1 + |Z|), is test_fast_normals_vs_oracle's)."""
    sl7 = gpu_lib
    torch = _torch()
    n_paths = 30_000 + 5
    ctx = sl7.Context(m)
    code = sl7.COLLOC_EXACT_GBM if colloc == "gbm" else sl7.COLLOC_EXACT_OU
    opts = sl7.make_opts(prec=sl7.PREC_FP32, colloc=code, flags=flags)
    out, _ = ctx.simulate(1.0, dt, n_steps, theta, n_paths, 77, sl7.OUT_FULL, opts)
    torch.cuda.synchronize()
    Yd = out.double().cpu().numpy().reshape(n_steps + 1, n_paths)
    spec = O.Spec(m, colloc, theta, 1.0, dt, n_steps)
    if flags & sl7.FLAG_FAST_NORMALS:
        z = torch.empty(n_steps * n_paths, dtype=torch.float32, device="cuda")
        sl7.normals(77, 0, n_paths, n_steps, z, flags=sl7.FLAG_FAST_NORMALS)
        torch.cuda.synchronize()
        Z = z.double().cpu().numpy().reshape(n_steps, n_paths)
    else:
        Z = O.normals(77, np.arange(n_paths, dtype=np.uint64), n_steps)
    worst = _teacher_forced(spec, Yd, Z)
    print("flags=%d worst |err|/kappa = %.3g" % (flags, worst))


@pytest.mark.parametrize("m,theta,n_steps,dt", [(5, (0.05, 0.2), 64, 1 / 64), (7, (0.05, 0.2), 6, 0.5),
                                                (6, (0.1, 0.5), 9, 0.25)])
def test_exact_full4_teacher_forced(gpu_lib, m, theta, n_steps, dt):
    """cfg3's FULL kernel (four paths per thread, 16-byte row stores, normals in units of sqrt(2 ln 2), Horner
    coefficients scaled by s^j; it runs when n_paths % 4 == 0): teacher-forced against the float64 oracle on
    the device's fast normals at 1e-5 * kappa, incl. m = 6 (padded Horner) and a 9-step tail of one block."""
    sl7 = gpu_lib
    torch = _torch()
    n_paths = 30_000
    ctx = sl7.Context(m)
    opts = sl7.make_opts(colloc=sl7.COLLOC_EXACT_GBM, flags=sl7.FLAG_FAST_NORMALS | sl7.FLAG_SPECIALIZED)
    out, _ = ctx.simulate(1.0, dt, n_steps, theta, n_paths, 78, sl7.OUT_FULL, opts)
    z = torch.empty(n_steps * n_paths, dtype=torch.float32, device="cuda")
    sl7.normals(78, 0, n_paths, n_steps, z, flags=sl7.FLAG_FAST_NORMALS)
    torch.cuda.synchronize()
    Yd = out.double().cpu().numpy().reshape(n_steps + 1, n_paths)
    Z = z.double().cpu().numpy().reshape(n_steps, n_paths)
    worst = _teacher_forced(O.Spec(m, "gbm", theta, 1.0, dt, n_steps), Yd, Z)
    print("full4 m=%d worst |err|/kappa = %.3g" % (m, worst))


def test_exact_full4_stats_and_reference(gpu_lib):
    """The FULL kernel's REF_ON form (FULL output + fused statistics + strong error against exact GBM on the
    same normals, which it rebuilds as -s W'): moments equal the oracle's statistics of the last row, the strong
    error stays at rounding level."""
    sl7 = gpu_lib
    torch = _torch()
    n_paths, n_steps, dt, theta = 40_000, 16, 1 / 16, (0.05, 0.2)
    ctx = sl7.Context(7)
    opts = sl7.make_opts(colloc=sl7.COLLOC_EXACT_GBM, flags=sl7.FLAG_FAST_NORMALS | sl7.FLAG_SPECIALIZED,
                         n_bins=256, hist_lo=0.0, hist_hi=3.0, shift=1.0, ref=sl7.REF_GBM, ref_theta=theta + (0,))
    st = torch.zeros(sl7.stats_elems(256), dtype=torch.float64, device="cuda")
    out, _ = ctx.simulate(1.0, dt, n_steps, theta, n_paths, 79, sl7.OUT_FULL, opts, stats=st)
    torch.cuda.synchronize()
    YT = out.double().cpu().numpy()[-n_paths:]
    v, s = O.stats_vector(YT, 1.0, 0.0, 3.0, 256), st.cpu().numpy()
    np.testing.assert_allclose(s[2:6], v[2:6], rtol=1e-12, atol=1e-9)
    assert s[8:].sum() == v[8:].sum() and np.abs(s[8:] - v[8:]).sum() <= 4   # T-5: edge ties only
    assert s[0] == n_paths and 0 < s[6] / s[0] < 2e-6


def test_fast_normals_vs_oracle(gpu_lib):
    """The SL7_FLAG_FAST_NORMALS Box-Muller (MUFU lg2 + series near u -> 1, MUFU sin/cos on the exactly
    reduced angle) stays within 2e-6 (1 + |Z|) of the float64 normals (measured 1.1e-6), including the
    u -> 1 tail."""
    torch = _torch()
    sl7 = gpu_lib
    n, steps, seed = 300_000, 8, 4242
    out = torch.empty(steps * n, dtype=torch.float32, device="cuda")
    sl7.normals(seed, 17, n, steps, out, flags=sl7.FLAG_FAST_NORMALS)
    torch.cuda.synchronize()
    dev = out.double().cpu().numpy().reshape(steps, n)
    ref = O.normals(seed, 17 + np.arange(n, dtype=np.uint64), steps)
    err = np.abs(dev - ref)
    assert np.all(err <= 2e-6 * (1.0 + np.abs(ref))), err.max()


@pytest.mark.parametrize("colloc,theta,ref", [("gbm", (0.05, 0.2), 1), ("ou", (0.0, 1.0, 0.5), 2)])
def test_specialized_stats_and_reference(gpu_lib, colloc, theta, ref):
    """Fused statistics and the strong-error reference in the specialised kernel (REF_ON variant):
    terminal values equal the FULL run's last row bitwise; moments match the oracle's statistics of
    those values; the strong error vs the exact solution on the same normals stays rounding-level."""
    sl7 = gpu_lib
    torch = _torch()
    n_paths, n_steps, dt = 50_001, 13, 1.0 / 13
    ctx = sl7.Context(7)
    code = sl7.COLLOC_EXACT_GBM if colloc == "gbm" else sl7.COLLOC_EXACT_OU
    flags = sl7.FLAG_FAST_NORMALS | sl7.FLAG_SPECIALIZED
    full, _ = ctx.simulate(1.0, dt, n_steps, theta, n_paths, 5, sl7.OUT_FULL, sl7.make_opts(colloc=code, flags=flags))
    YT, st = _run(sl7, ctx, dict(y0=1.0, dt=dt, n_steps=n_steps), n_paths, 5, sl7.OUT_TERMINAL, code, stats=True,
                  n_bins=256, lo=-2.0, hi=3.0, shift=1.0, ref=ref, ref_theta=theta + (0,) * (3 - len(theta)),
                  theta=theta, flags=flags)
    torch.cuda.synchronize()
    assert np.array_equal(full.double().cpu().numpy()[-n_paths:], YT)
    v = O.stats_vector(YT, 1.0, -2.0, 3.0, 256)
    np.testing.assert_allclose(st[2:6], v[2:6], rtol=1e-12, atol=1e-9)
    assert st[0] == n_paths and st[6] / st[0] < 2e-6


def test_specialized_rejects_large_m(gpu_lib):
    sl7 = gpu_lib
    ctx = sl7.Context(9)
    opts = sl7.make_opts(colloc=sl7.COLLOC_EXACT_GBM, flags=sl7.FLAG_SPECIALIZED)
    with pytest.raises(sl7.Sl7Error, match="EUNSUPPORTED"):
        ctx.simulate(1.0, 0.5, 2, (0.05, 0.2), 100, 1, sl7.OUT_TERMINAL, opts)


@pytest.mark.parametrize("prec", ["fp32", "split"])
def test_multistep_ann_affine_network_free_running(gpu_lib, prec):
    """16 free-running ANN steps of the exactly-affine softplus network (tests/test_oracle_pins.py) against
    the closed-form recursion Y <- a32 Y + L(Z) on the device's own normals: fp32-class kernels stay within
    the accumulated activation error (4 layers x 2 units x ~2.5e-7 per step, ~16 steps)."""
    from _helpers import affine_softplus_mlp
    sl7 = gpu_lib
    torch = _torch()
    theta, dt, n, m, N = (0.3, 1.2, 0.4), 0.125, 16, 7, 20_000
    ybar, lam, sig = theta
    x = O.gauss_hermite_nodes(m)
    a = np.exp(-lam * dt)
    b = ybar * (1 - a)
    s = sig * np.sqrt((1 - np.exp(-2 * lam * dt)) / (2 * lam))
    blob = pack_blob(affine_softplus_mlp((5, 50, 50, 50, 50, m), a, b + s * x))
    ctx = sl7.Context(m, [5, 50, 50, 50, 50, m], ACT_SOFTPLUS)
    ctx.load_weights(blob)
    p = {"fp32": sl7.PREC_FP32, "split": sl7.PREC_SPLIT}[prec]
    out, _ = ctx.simulate(0.7, dt, n, theta, N, 21, sl7.OUT_FULL, sl7.make_opts(prec=p, colloc=sl7.COLLOC_ANN))
    z = torch.empty(n * N, dtype=torch.float32, device="cuda")
    sl7.normals(21, 0, N, n, z)
    torch.cuda.synchronize()
    Yd = out.double().cpu().numpy().reshape(n + 1, N)
    Z = z.double().cpu().numpy().reshape(n, N)
    a32 = float(np.float32(a))
    c32 = (b + s * x).astype(np.float32).astype(np.float64)
    Y = np.full(N, float(np.float32(0.7)))
    for i in range(n):
        Y = a32 * Y + O.lagrange_eval(Z[i], x, np.broadcast_to(c32, (N, m)))
        assert np.abs(Yd[i + 1] - Y).max() <= 5e-6 * (i + 1), (i, np.abs(Yd[i + 1] - Y).max())


@pytest.mark.parametrize("m", [1, 2, 3, 16])
@pytest.mark.parametrize("kind", ["exact", "fp32", "bf16", "tf32", "split", "cdc"])
def test_edge_node_counts(gpu_lib, m, kind):
    """m = 1 (g_m is the constant y_0: the conditional median, no randomness), m = 2, 3, and the largest
    grid m = 16 (a 64-wide network, runtime-m kernels) for every kernel family, teacher-forced."""
    sl7 = gpu_lib
    n_paths, n_steps, dt = 3 * 128 + 5, 3, 0.25
    if kind == "exact":
        ctx = sl7.Context(m)
        colloc, prec, theta, quant, oc = sl7.COLLOC_EXACT_GBM, sl7.PREC_FP32, (0.05, 0.2), None, "gbm"
        spec = O.Spec(m, "gbm", theta, 1.0, dt, n_steps)
    else:
        dims = [4, 64, 64, m]
        p = glorot_mlp(dims, ACT_TANH, seed=5, with_norm=True)
        blob = pack_blob(p)
        ctx = sl7.Context(m, dims, ACT_TANH)
        ctx.load_weights(blob)
        theta = (0.3, 0.5)
        prec = {"fp32": sl7.PREC_FP32, "bf16": sl7.PREC_BF16, "tf32": sl7.PREC_TF32, "split": sl7.PREC_SPLIT,
                "cdc": sl7.PREC_FP32}[kind]
        quant = kind if kind in ("bf16", "tf32") else None
        colloc = sl7.COLLOC_ANN
        spec = O.Spec(m, "ann", theta, 1.0, dt, n_steps, net=O.parse_blob(blob), quant=quant)
    scheme = sl7.SCHEME_CDC if kind == "cdc" else sl7.SCHEME_7L
    torch = _torch()
    opts = sl7.make_opts(prec=prec, colloc=colloc, scheme=scheme)
    out, _ = ctx.simulate(1.0, dt, n_steps, theta, n_paths, 13, sl7.OUT_FULL, opts)
    torch.cuda.synchronize()
    Yd = out.double().cpu().numpy().reshape(n_steps + 1, n_paths)
    Z = O.normals(13, np.arange(n_paths, dtype=np.uint64), n_steps)
    tol = 5e-3 if quant else 1e-5
    for i in range(n_steps):
        if kind == "cdc":
            ref, kap = O.cdc_step(spec, Yd[i], Z[i]), O.cdc_step_error_scale(spec, Yd[i], Z[i])
        else:
            ref, kap = O.step(spec, Yd[i], Z[i]), O.step_error_scale(spec, Yd[i], Z[i])
        r = np.abs(Yd[i + 1] - ref) / kap
        assert r.max() <= tol, (kind, m, i, float(r.max()))
    if m == 1 and kind == "exact":   # no randomness: Y0 c_0^i with c_0 = exp((mu - s^2/2) dt)
        c0 = np.float32(np.exp((0.05 - 0.02) * dt))
        assert np.all(np.abs(Yd[-1] - float(c0) ** n_steps) <= 1e-6)
