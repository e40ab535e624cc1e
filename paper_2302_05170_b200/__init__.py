"""Python binding of libsl7.so, the B200-native Seven-League online path generator.

Argument marshalling only (ctypes): every step of the path runs inside the library's CUDA kernels.
Names follow include/sl7.h.  PyTorch provides device memory and streams; there is NO CPU fallback --
if the library or a CUDA device is missing, calls raise.

    import paper_2302_05170_b200 as sl7
    ctx = sl7.Context(m=7, layer_dims=[2, 50, 50, 50, 7], act=sl7.ACT_TANH)
    ctx.load_weights(blob)
    out, stats = ctx.simulate(y0=1.0, dt=1/64, n_steps=64, theta=(), n_paths=10**7, seed=1,
                              out_mode=sl7.OUT_STATS, prec=sl7.PREC_FP32, n_bins=4096, ...)
"""
from __future__ import annotations

import ctypes
import os

PKG = os.path.dirname(os.path.abspath(__file__))
# SL7_LIB: an experiment build (python -m paper_2302_05170_b200.build --ab -> libsl7_ab.so) for A/B timings
LIB_PATH = os.environ.get("SL7_LIB") or os.path.join(PKG, "libsl7.so")

OK, EINVAL, ESTATE, EFORMAT, ENOMEM, ECUDA, ENONFINITE, EUNSUPPORTED = range(8)
ACT_TANH, ACT_SOFTPLUS = 0, 1
OUT_FULL, OUT_TERMINAL, OUT_STATS = 0, 1, 2
PREC_FP32, PREC_TF32, PREC_BF16, PREC_SPLIT = 0, 1, 2, 3
COLLOC_ANN, COLLOC_EXACT_GBM, COLLOC_EXACT_OU, COLLOC_EXACT_CIR = 0, 1, 2, 3
REF_NONE, REF_GBM, REF_OU = 0, 1, 2
MODEL_GBM, MODEL_OU, MODEL_CIR = 1, 2, 3
STATS_HEAD = 8
MAX_M = 16
HAS_TC = True   # libsl7 has the tcgen05 (SL7_PREC_BF16) ANN kernel


class sl7_run_opts(ctypes.Structure):
    _fields_ = [("prec", ctypes.c_int), ("colloc", ctypes.c_int), ("path_offset", ctypes.c_uint64),
                ("stream", ctypes.c_void_p), ("hist_lo", ctypes.c_double), ("hist_hi", ctypes.c_double),
                ("shift", ctypes.c_double), ("n_bins", ctypes.c_int32), ("accumulate", ctypes.c_int32),
                ("ref", ctypes.c_int), ("ref_theta", ctypes.c_double * 3), ("flags", ctypes.c_uint32),
                ("scheme", ctypes.c_int)]


SCHEME_7L, SCHEME_CDC, SCHEME_CDC_PRED = 0, 1, 2


FLAG_FAST_NORMALS = 1
FLAG_SPECIALIZED = 2


class sl7_summary(ctypes.Structure):
    _fields_ = [("n", ctypes.c_uint64), ("n_nonfinite", ctypes.c_uint64), ("mean", ctypes.c_double),
                ("var", ctypes.c_double), ("skew", ctypes.c_double), ("exkurt", ctypes.c_double),
                ("strong_err", ctypes.c_double), ("rms_err", ctypes.c_double),
                ("q_levels", ctypes.POINTER(ctypes.c_double)), ("q_values", ctypes.POINTER(ctypes.c_double)),
                ("n_q", ctypes.c_int32)]


class Sl7Error(RuntimeError):
    def __init__(self, status, msg):
        super().__init__("%s: %s" % (STATUS_NAMES.get(status, status), msg))
        self.status = status


STATUS_NAMES = {0: "SL7_OK", 1: "SL7_EINVAL", 2: "SL7_ESTATE", 3: "SL7_EFORMAT", 4: "SL7_ENOMEM",
                5: "SL7_ECUDA", 6: "SL7_ENONFINITE", 7: "SL7_EUNSUPPORTED"}

EXPORTS = ["sl7_create", "sl7_load_weights", "sl7_simulate", "sl7_simulate_host", "sl7_simulate_host_async",
           "sl7_sync", "sl7_simulate_em",
           "sl7_training_set", "sl7_cdc_hist_elems", "sl7_cdc_init", "sl7_cdc_hist", "sl7_cdc_select",
           "sl7_cdc_step", "sl7_stats",
           "sl7_philox_u32", "sl7_normals", "sl7_gh_grid", "sl7_out_elems", "sl7_stats_elems",
           "sl7_last_error", "sl7_status_str", "sl7_abi_version", "sl7_destroy"]

_lib = None


def load_library(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load libsl7.so (raises if it has not been built: there is no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError("libsl7.so not built (run python -m paper_2302_05170_b200.build): %s" % path)
    L = ctypes.CDLL(path)
    c = ctypes
    u64, i32, vp, dp, fp = c.c_uint64, c.c_int32, c.c_void_p, c.POINTER(c.c_double), c.c_void_p
    L.sl7_create.argtypes = [i32, c.POINTER(i32), i32, c.c_int, i32, c.POINTER(vp)]
    L.sl7_load_weights.argtypes = [vp, c.c_char_p, c.c_size_t]
    L.sl7_simulate.argtypes = [vp, c.c_double, c.c_double, i32, dp, i32, u64, u64, c.c_int,
                               c.POINTER(sl7_run_opts), fp, fp]
    L.sl7_simulate_host.argtypes = [vp, c.c_double, c.c_double, i32, dp, i32, u64, u64, c.c_int,
                                    c.POINTER(sl7_run_opts), fp, fp, c.POINTER(u64), c.POINTER(u64)]
    L.sl7_simulate_host_async.argtypes = L.sl7_simulate_host.argtypes
    L.sl7_sync.argtypes = [vp]
    L.sl7_simulate_em.argtypes = [vp, c.c_int, c.c_double, c.c_double, i32, i32, dp, i32, u64, u64, c.c_int,
                                  c.POINTER(sl7_run_opts), fp, fp]
    L.sl7_training_set.argtypes = [vp, c.c_int, dp, u64, c.c_uint32, c.c_double, u64, c.POINTER(sl7_run_opts),
                                   fp, fp]
    L.sl7_cdc_hist_elems.argtypes = []
    L.sl7_cdc_hist_elems.restype = c.c_size_t
    L.sl7_cdc_init.argtypes = [vp, c.c_double, c.c_double, i32, dp, i32, u64, u64, c.POINTER(sl7_run_opts), fp]
    L.sl7_cdc_hist.argtypes = [vp, fp, i32, fp]
    L.sl7_cdc_select.argtypes = [vp, i32, fp]
    L.sl7_cdc_step.argtypes = [vp, i32, fp, fp, fp]
    L.sl7_stats.argtypes = [dp, c.POINTER(sl7_run_opts), c.POINTER(sl7_summary)]
    L.sl7_philox_u32.argtypes = [u64, u64, u64, c.c_uint32, vp, vp]
    L.sl7_normals.argtypes = [u64, u64, u64, i32, c.c_uint32, vp, vp]
    L.sl7_gh_grid.argtypes = [i32, dp, dp]
    L.sl7_out_elems.argtypes = [i32, u64, c.c_int]
    L.sl7_out_elems.restype = c.c_size_t
    L.sl7_stats_elems.argtypes = [i32]
    L.sl7_stats_elems.restype = c.c_size_t
    L.sl7_last_error.argtypes = [vp]
    L.sl7_last_error.restype = c.c_char_p
    L.sl7_status_str.argtypes = [c.c_int]
    L.sl7_status_str.restype = c.c_char_p
    L.sl7_abi_version.restype = i32
    L.sl7_destroy.argtypes = [vp]
    L.sl7_destroy.restype = None
    for name in ("sl7_create", "sl7_load_weights", "sl7_simulate", "sl7_simulate_host", "sl7_simulate_host_async",
                 "sl7_sync", "sl7_simulate_em",
                 "sl7_training_set", "sl7_cdc_init", "sl7_cdc_hist", "sl7_cdc_select", "sl7_cdc_step", "sl7_stats",
                 "sl7_philox_u32", "sl7_normals", "sl7_gh_grid"):
        getattr(L, name).restype = c.c_int
    _lib = L
    return L


def _check(st, ctx=None):
    if st != OK:
        msg = _lib.sl7_last_error(ctx).decode()
        raise Sl7Error(st, msg)


def _dptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _dbuf(t, dtype, n, name):
    """Device pointer of a caller tensor after checking what the C ABI cannot: a contiguous CUDA tensor of
    the expected dtype holding at least n elements (the library writes n of them)."""
    if t is None:
        return None
    import torch
    if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == dtype and t.is_contiguous()):
        raise Sl7Error(EINVAL, "%s must be a contiguous CUDA %s tensor" % (name, dtype))
    if n is not None and t.numel() < n:
        raise Sl7Error(EINVAL, "%s holds %d elements, %d needed" % (name, t.numel(), n))
    return ctypes.c_void_p(t.data_ptr())


def _stream_ptr(stream):
    import torch
    s = torch.cuda.current_stream() if stream is None else stream
    return ctypes.c_void_p(s.cuda_stream)


def make_opts(prec=PREC_FP32, colloc=COLLOC_ANN, path_offset=0, stream=None, hist_lo=0.0, hist_hi=0.0,
              shift=0.0, n_bins=0, accumulate=0, ref=REF_NONE, ref_theta=(0.0, 0.0, 0.0), raw_stream=None,
              flags=0, scheme=SCHEME_7L):
    o = sl7_run_opts()
    o.prec, o.colloc, o.path_offset, o.flags, o.scheme = prec, colloc, int(path_offset), int(flags), int(scheme)
    o.stream = raw_stream if raw_stream is not None else (_stream_ptr(stream) if stream is not False else None)
    o.hist_lo, o.hist_hi, o.shift, o.n_bins, o.accumulate = hist_lo, hist_hi, shift, int(n_bins), int(accumulate)
    o.ref = ref
    for k in range(3):
        o.ref_theta[k] = float(ref_theta[k]) if k < len(ref_theta) else 0.0
    return o


def gh_grid(m: int):
    """Host-setup nodes and barycentric weights (double) as computed inside the library."""
    L = load_library()
    x = (ctypes.c_double * m)()
    w = (ctypes.c_double * m)()
    _check(L.sl7_gh_grid(m, x, w))
    return list(x), list(w)


def out_elems(n_steps, n_paths, mode):
    return load_library().sl7_out_elems(n_steps, n_paths, mode)


def stats_elems(n_bins):
    return load_library().sl7_stats_elems(n_bins)


def stats_summary(h_stats, opts, q_levels=()):
    """Moments / strong error / histogram quantiles of a host stats vector (list, numpy or tensor)."""
    L = load_library()
    import numpy as np
    v = np.ascontiguousarray(np.asarray(h_stats, dtype=np.float64))
    s = sl7_summary()
    lv = (ctypes.c_double * max(1, len(q_levels)))(*q_levels)
    qv = (ctypes.c_double * max(1, len(q_levels)))()
    s.q_levels, s.q_values, s.n_q = lv, qv, len(q_levels)
    st = L.sl7_stats(v.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), ctypes.byref(opts), ctypes.byref(s))
    if st not in (OK, ENONFINITE):
        _check(st)
    out = {"n": s.n, "n_nonfinite": s.n_nonfinite, "mean": s.mean, "var": s.var, "skew": s.skew,
           "exkurt": s.exkurt, "strong_err": s.strong_err, "rms_err": s.rms_err,
           "quantiles": [qv[i] for i in range(len(q_levels))], "status": st}
    if opts.scheme == SCHEME_CDC_PRED:
        # E1 of a CDC_PRED run counts the path-steps clamped to the marginal hull (include/sl7.h)
        out["clamped_steps"] = float(v[6])
        out["strong_err"] = out["rms_err"] = 0.0
    return out


def philox_u32(seed, path_offset, n_paths, block, out, stream=None):
    L = load_library()
    import torch
    o = _dbuf(out, out.dtype if out is not None and out.dtype in (torch.int32, torch.uint32) else torch.int32, 4 * int(n_paths), "out")
    _check(L.sl7_philox_u32(int(seed), int(path_offset), int(n_paths), int(block), o, _stream_ptr(stream)))
    return out


def normals(seed, path_offset, n_paths, n_steps, out, stream=None, flags=0):
    L = load_library()
    import torch
    o = _dbuf(out, torch.float32, int(n_paths) * int(n_steps), "out")
    _check(L.sl7_normals(int(seed), int(path_offset), int(n_paths), int(n_steps), int(flags), o,
                         _stream_ptr(stream)))
    return out


_LIVE = None   # weak set of open contexts, closed at interpreter exit (before the CUDA runtime is torn down)


def _close_all():
    for c in list(_LIVE or ()):
        c.close()


class Context:
    """Owns one sl7_ctx (one device)."""

    def __init__(self, m, layer_dims=None, act=ACT_TANH, device=None):
        import torch
        L = load_library()
        self.device = torch.cuda.current_device() if device is None else int(device)
        self.m = m
        dims = list(layer_dims or [])
        arr = (ctypes.c_int32 * max(1, len(dims)))(*dims)
        h = ctypes.c_void_p()
        _check(L.sl7_create(m, arr if dims else None, len(dims), act, self.device, ctypes.byref(h)))
        self._h = h
        self.layer_dims = dims
        global _LIVE
        if _LIVE is None:
            import atexit
            import weakref
            _LIVE = weakref.WeakSet()
            atexit.register(_close_all)
        _LIVE.add(self)

    def close(self):
        h = getattr(self, "_h", None)
        if h and _lib is not None:      # at interpreter exit the module global may already be gone
            _lib.sl7_destroy(h)
        self._h = None

    __del__ = close

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()
        return False

    def load_weights(self, blob: bytes):
        _check(_lib.sl7_load_weights(self._h, blob, len(blob)), self._h)

    def simulate(self, y0, dt, n_steps, theta, n_paths, seed, out_mode, opts, out=None, stats=None):
        """sl7_simulate on torch device tensors (float32 out, float64 stats); allocates if None."""
        import torch
        dev = torch.device("cuda", self.device)
        if out is None and out_mode != OUT_STATS:
            out = torch.empty(out_elems(n_steps, n_paths, out_mode), dtype=torch.float32, device=dev)
        th = (ctypes.c_double * max(1, len(theta)))(*theta)
        po = _dbuf(out, torch.float32, out_elems(n_steps, n_paths, out_mode), "out") if out_mode != OUT_STATS else None
        ps = _dbuf(stats, torch.float64, _stats_need(opts), "stats")
        _check(_lib.sl7_simulate(self._h, float(y0), float(dt), int(n_steps), th, len(theta), int(n_paths),
                                 int(seed), out_mode, ctypes.byref(opts), po, ps), self._h)
        return out, stats

    def simulate_host(self, y0, dt, n_steps, theta, n_paths, seed, out_mode, opts, h_out=None, h_stats=None):
        """sl7_simulate_host on host numpy buffers; returns (h_out, h_stats, h2d_bytes, d2h_bytes)."""
        import numpy as np
        th = (ctypes.c_double * max(1, len(theta)))(*theta)
        up, down = ctypes.c_uint64(), ctypes.c_uint64()
        def hbuf(a, dtype, n, name):
            if a is None:
                return None
            if not (isinstance(a, np.ndarray) and a.dtype == dtype and a.flags["C_CONTIGUOUS"] and a.size >= n):
                raise Sl7Error(EINVAL, "%s must be a C-contiguous numpy %s array of >= %d elements" % (name, dtype, n))
            return a.ctypes.data_as(ctypes.c_void_p)
        po = hbuf(h_out, np.float32, out_elems(n_steps, n_paths, out_mode), "h_out") if out_mode != OUT_STATS else None
        ps = hbuf(h_stats, np.float64, _stats_need(opts) or 0, "h_stats")
        _check(_lib.sl7_simulate_host(self._h, float(y0), float(dt), int(n_steps), th, len(theta), int(n_paths),
                                      int(seed), out_mode, ctypes.byref(opts), po, ps, ctypes.byref(up),
                                      ctypes.byref(down)), self._h)
        return h_out, h_stats, up.value, down.value

    def simulate_host_async(self, y0, dt, n_steps, theta, n_paths, seed, out_mode, opts, h_out=None, h_stats=None):
        """sl7_simulate_host_async: enqueue a host-buffer run and return (h_out, h_stats, h2d, d2h) at once;
        the buffers (ideally pinned) hold the results after sync()."""
        import numpy as np
        th = (ctypes.c_double * max(1, len(theta)))(*theta)
        up, down = ctypes.c_uint64(), ctypes.c_uint64()

        def hbuf(a, dtype, n, name):
            if a is None:
                return None
            if not (isinstance(a, np.ndarray) and a.dtype == dtype and a.flags["C_CONTIGUOUS"] and a.size >= n):
                raise Sl7Error(EINVAL, "%s must be a C-contiguous numpy %s array of >= %d elements" % (name, dtype, n))
            return a.ctypes.data_as(ctypes.c_void_p)
        po = hbuf(h_out, np.float32, out_elems(n_steps, n_paths, out_mode), "h_out") if out_mode != OUT_STATS else None
        ps = hbuf(h_stats, np.float64, _stats_need(opts) or 0, "h_stats")
        _check(_lib.sl7_simulate_host_async(self._h, float(y0), float(dt), int(n_steps), th, len(theta), int(n_paths),
                                            int(seed), out_mode, ctypes.byref(opts), po, ps, ctypes.byref(up),
                                            ctypes.byref(down)), self._h)
        return h_out, h_stats, up.value, down.value

    def sync(self):
        _check(_lib.sl7_sync(self._h), self._h)

    def simulate_em(self, model, y0, dt, n_steps, substeps, theta, n_paths, seed, out_mode, opts, out=None,
                    stats=None):
        """sl7_simulate_em (Euler-Maruyama comparator) on torch device tensors; allocates out if None."""
        import torch
        dev = torch.device("cuda", self.device)
        if out is None and out_mode != OUT_STATS:
            out = torch.empty(out_elems(n_steps, n_paths, out_mode), dtype=torch.float32, device=dev)
        th = (ctypes.c_double * max(1, len(theta)))(*theta)
        po = _dbuf(out, torch.float32, out_elems(n_steps, n_paths, out_mode), "out") if out_mode != OUT_STATS else None
        ps = _dbuf(stats, torch.float64, _stats_need(opts), "stats")
        _check(_lib.sl7_simulate_em(self._h, int(model), float(y0), float(dt), int(n_steps), int(substeps), th,
                                    len(theta), int(n_paths), int(seed), out_mode, ctypes.byref(opts), po, ps), self._h)
        return out, stats

    def training_set(self, model, features, n_inner, dtau, seed, opts, terminal=None, labels=None):
        """sl7_training_set: features = host float64 [n_rows][2 + n_theta]; returns (terminal, labels) device
        tensors (terminal None unless passed in: the library then uses its own scratch)."""
        import numpy as np
        import torch
        F = np.ascontiguousarray(np.asarray(features, dtype=np.float64))
        n_rows = F.shape[0]
        if labels is None:
            labels = torch.empty((n_rows, self.m), dtype=torch.float64, device=torch.device("cuda", self.device))
        pt = _dbuf(terminal, torch.float32, n_rows * int(n_inner), "terminal")
        pl = _dbuf(labels, torch.float64, n_rows * self.m, "labels")
        _check(_lib.sl7_training_set(self._h, int(model), F.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                     int(n_rows), int(n_inner), float(dtau), int(seed), ctypes.byref(opts),
                                     pt, pl), self._h)
        return terminal, labels

    # ---- sharded 7L-CDC (include/sl7.h, "Sharded 7L-CDC"): the caller drives the loop -------------
    def cdc_init(self, y0, dt, n_steps, theta, n_paths, seed, opts, state):
        import torch
        th = (ctypes.c_double * max(1, len(theta)))(*theta)
        ps = _dbuf(state, torch.float32, int(n_paths), "state")
        _check(_lib.sl7_cdc_init(self._h, float(y0), float(dt), int(n_steps), th, len(theta), int(n_paths), int(seed),
                                 ctypes.byref(opts), ps), self._h)
        self._cdc_n, self._cdc_bins = int(n_paths), int(opts.n_bins)

    def cdc_hist(self, state, pass_, hist):
        import torch
        n = getattr(self, "_cdc_n", 0)
        _check(_lib.sl7_cdc_hist(self._h, _dbuf(state, torch.float32, n, "state"), int(pass_),
                                 _dbuf(hist, torch.int64, cdc_hist_elems(), "hist")), self._h)

    def cdc_select(self, pass_, hist):
        import torch
        _check(_lib.sl7_cdc_select(self._h, int(pass_), _dbuf(hist, torch.int64, cdc_hist_elems(), "hist")), self._h)

    def cdc_step(self, step, state_in, state_out, stats=None):
        import torch
        n = getattr(self, "_cdc_n", 0)
        _check(_lib.sl7_cdc_step(self._h, int(step), _dbuf(state_in, torch.float32, n, "state_in"),
                                 _dbuf(state_out, torch.float32, n, "state_out"),
                                 _dbuf(stats, torch.float64, stats_elems(getattr(self, "_cdc_bins", 0)), "stats")),
               self._h)


def _stats_need(opts):
    """Elements of the stats vector opts describes (None when n_bins is invalid: the library rejects it)."""
    return stats_elems(opts.n_bins) if 0 <= opts.n_bins <= 16384 else None


def cdc_hist_elems():
    return load_library().sl7_cdc_hist_elems()
