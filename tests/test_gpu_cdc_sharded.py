"""Sharded 7L-CDC through sl7_cdc_init/hist/select/step (include/sl7.h "Sharded 7L-CDC") on one GPU:
one shard equals sl7_simulate(scheme = CDC) bit for bit; two shards of one process (two contexts, the
histograms summed as the all-reduce would) equal the single run over the union of their paths, per path
bit for bit, with the same histogram counts and moments within 1e-12 (T-6)."""
import numpy as np
import pytest

from sl7_inputs import load_golden_blob, workloads

pytestmark = pytest.mark.gpu


def _torch():
    import torch
    return torch


def _setup(sl7, kind):
    w = workloads()["cfg2_ou"]
    if kind == "exact":
        ctxs = [sl7.Context(w.m) for _ in range(2)]
        colloc, prec = sl7.COLLOC_EXACT_OU, sl7.PREC_FP32
    else:
        ctxs = [sl7.Context(w.m, list(w.dims), w.act) for _ in range(2)]
        for c in ctxs:
            c.load_weights(load_golden_blob(w.blob))
        colloc, prec = sl7.COLLOC_ANN, sl7.PREC_FP32
    return w, ctxs, colloc, prec


@pytest.mark.parametrize("kind", ["exact", "ann"])
def test_sharded_cdc_equals_single_run(gpu_lib, kind):
    sl7 = gpu_lib
    torch = _torch()
    from paper_2302_05170_b200.dist import CdcShard, cdc_run
    w, ctxs, colloc, prec = _setup(sl7, kind)
    n_steps, N1, N2, nb = 6, 37_001, 20_555, 128
    N = N1 + N2
    kw = dict(prec=prec, colloc=colloc, scheme=sl7.SCHEME_CDC, n_bins=nb, hist_lo=-3.0, hist_hi=3.0, shift=1.0)
    # reference: one sl7_simulate call over all N paths
    ref_st = torch.zeros(sl7.stats_elems(nb), dtype=torch.float64, device="cuda")
    ref, _ = ctxs[0].simulate(w.y0, w.dt, n_steps, w.theta, N, w.seed, sl7.OUT_TERMINAL, sl7.make_opts(**kw),
                              stats=ref_st)
    # one shard through the split API
    st1 = torch.zeros_like(ref_st)
    (s,) = cdc_run([CdcShard(ctxs[0], w.y0, w.dt, n_steps, w.theta, N, w.seed, sl7.make_opts(**kw), st1)], n_steps)
    torch.cuda.synchronize()
    assert torch.equal(s.state, ref)
    r, v = ref_st.cpu().numpy(), st1.cpu().numpy()          # fp64 atomics: summation order may differ
    assert r[0] == v[0] == N and np.array_equal(r[8:], v[8:])
    np.testing.assert_allclose(v[2:6], r[2:6], rtol=1e-12)
    # two shards: paths [0, N1) and [N1, N)
    st2 = torch.zeros_like(ref_st)
    a = CdcShard(ctxs[0], w.y0, w.dt, n_steps, w.theta, N1, w.seed, sl7.make_opts(path_offset=0, **kw), st2)
    b = CdcShard(ctxs[1], w.y0, w.dt, n_steps, w.theta, N2, w.seed, sl7.make_opts(path_offset=N1, **kw), st2)
    cdc_run([a, b], n_steps)
    torch.cuda.synchronize()
    assert torch.equal(torch.cat([a.state, b.state]), ref)
    r, v = ref_st.cpu().numpy(), st2.cpu().numpy()
    assert r[0] == v[0] == N and np.array_equal(r[8:], v[8:])
    np.testing.assert_allclose(v[2:6], r[2:6], rtol=1e-12)


def test_sharded_cdc_api_errors(gpu_lib):
    sl7 = gpu_lib
    torch = _torch()
    ctx = sl7.Context(5)
    h = torch.zeros(sl7.cdc_hist_elems(), dtype=torch.int64, device="cuda")
    y = torch.zeros(10, dtype=torch.float32, device="cuda")
    with pytest.raises(sl7.Sl7Error, match="ESTATE"):
        ctx.cdc_hist(y, 0, h)
    o = sl7.make_opts(colloc=sl7.COLLOC_EXACT_GBM, scheme=sl7.SCHEME_CDC)
    ctx.cdc_init(1.0, 0.5, 2, (0.05, 0.2), 10, 1, o, y)
    with pytest.raises(sl7.Sl7Error, match="pass"):
        ctx.cdc_hist(y, 4, h)
    with pytest.raises(sl7.Sl7Error, match="step"):
        ctx.cdc_step(2, y, y)
    with pytest.raises(sl7.Sl7Error, match="ref"):
        ctx.cdc_init(1.0, 0.5, 2, (0.05, 0.2), 10, 1,
                     sl7.make_opts(colloc=sl7.COLLOC_EXACT_GBM, ref=sl7.REF_GBM, ref_theta=(0.05, 0.2)), y)
