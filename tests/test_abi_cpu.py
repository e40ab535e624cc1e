"""C-ABI library on the CPU box: it loads, exports every entry point include/sl7.h declares, and its
host-side logic (grid setup, argument validation, statistics summary) is right.  No compute call is
made here (no GPU): compute entry points must fail loudly with SL7_ECUDA, never fall back."""
import ctypes
import math
import os
import re
import subprocess

import numpy as np
import pytest

import paper_2302_05170_b200 as sl7
from oracle import sl7_oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "sl7.h")


@pytest.fixture(scope="module")
def lib():
    from paper_2302_05170_b200 import build
    build.build(verbose=False)
    return sl7.load_library()


def declared_functions():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(sl7_[a-z0-9_]+)\s*\(", txt)))


def test_exports_every_declared_symbol(lib):
    names = declared_functions()
    assert len(names) >= 14
    out = subprocess.run(["nm", "-D", "--defined-only", sl7.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (sl7_\w+)", out))
    missing = [n for n in names if n not in exported]
    assert not missing, missing
    assert set(names) == set(sl7.EXPORTS)
    for n in names:
        getattr(lib, n)


def test_library_is_sm100a(lib):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", sl7.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_abi_version_and_sizes(lib):
    assert lib.sl7_abi_version() == 2
    assert lib.sl7_out_elems(64, 1000, sl7.OUT_FULL) == 65 * 1000
    assert lib.sl7_out_elems(64, 1000, sl7.OUT_TERMINAL) == 1000
    assert lib.sl7_out_elems(64, 1000, sl7.OUT_STATS) == 0
    assert lib.sl7_stats_elems(4096) == 8 + 4096 + 2
    assert lib.sl7_stats_elems(0) == 10
    assert lib.sl7_status_str(6) == b"SL7_ENONFINITE"


@pytest.mark.parametrize("m", range(1, 17))
def test_host_grid_matches_oracle_and_closed_forms(lib, m):
    x, w = sl7.gh_grid(m)
    np.testing.assert_allclose(x, O.gauss_hermite_nodes(m), atol=2e-15 * max(1, m))
    np.testing.assert_allclose(w, O.bary_weights(O.gauss_hermite_nodes(m)), rtol=1e-13)
    assert x == [-v for v in x[::-1]]       # symmetric by construction


def test_grid_rejects_bad_m(lib):
    x = (ctypes.c_double * 20)()
    assert lib.sl7_gh_grid(0, x, x) == sl7.EINVAL
    assert lib.sl7_gh_grid(17, x, x) == sl7.EINVAL
    assert b"m must be" in lib.sl7_last_error(None)


def test_create_validates_before_touching_device(lib):
    h = ctypes.c_void_p()
    dims = (ctypes.c_int32 * 5)(2, 50, 50, 50, 5)
    assert lib.sl7_create(0, dims, 5, 0, 0, ctypes.byref(h)) == sl7.EINVAL
    assert lib.sl7_create(7, dims, 5, 0, 0, ctypes.byref(h)) == sl7.EINVAL      # last dim != m
    assert b"layer_dims" in lib.sl7_last_error(None)
    bad = (ctypes.c_int32 * 5)(2, 50, 65, 50, 5)
    assert lib.sl7_create(5, bad, 5, 0, 0, ctypes.byref(h)) == sl7.EINVAL
    assert lib.sl7_create(5, dims, 5, 3, 0, ctypes.byref(h)) == sl7.EINVAL      # act


def test_no_cpu_fallback(lib):
    """Without a device every compute path reports SL7_ECUDA instead of computing on the CPU."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("box has a GPU")
    h = ctypes.c_void_p()
    dims = (ctypes.c_int32 * 5)(2, 50, 50, 50, 5)
    assert lib.sl7_create(5, dims, 5, 0, 0, ctypes.byref(h)) == sl7.ECUDA
    assert lib.sl7_philox_u32(1, 0, 16, 0, ctypes.c_void_p(0x1000), None) != sl7.OK
    with pytest.raises(sl7.Sl7Error):
        sl7.Context(5, [2, 50, 50, 50, 5], device=0)


def _opts(n_bins, lo, hi, shift):
    return sl7.make_opts(stream=False, n_bins=n_bins, hist_lo=lo, hist_hi=hi, shift=shift)


def test_stats_summary_matches_oracle(lib):
    rng = np.random.default_rng(4)
    y = rng.lognormal(0.05, 0.2, 200_001)
    ref = y * (1 + 1e-4 * rng.normal(size=y.size))
    v = O.stats_vector(y, 1.0, 0.0, 3.0, 4096, ref)
    s = sl7.stats_summary(v, _opts(4096, 0.0, 3.0, 1.0), q_levels=[0.01, 0.25, 0.5, 0.75, 0.99])
    mo = O.moments_from_stats(v, 1.0)
    assert s["status"] == sl7.OK and s["n"] == y.size
    for k in ("mean", "var", "skew", "exkurt", "strong_err", "rms_err"):
        assert abs(s[k] - mo[k]) <= 1e-12 * max(1.0, abs(mo[k])), k
    qo = O.quantiles(y, [0.01, 0.25, 0.5, 0.75, 0.99])
    w = 3.0 / 4096
    assert np.all(np.abs(np.array(s["quantiles"]) - qo) <= w)     # T-5: within one bin width


def test_stats_nonfinite_and_empty(lib):
    y = np.array([1.0, 2.0, np.nan, np.inf])
    v = O.stats_vector(y, 0.0, 0.0, 4.0, 4)
    s = sl7.stats_summary(v, _opts(4, 0.0, 4.0, 0.0))
    assert s["status"] == sl7.ENONFINITE and s["n"] == 2 and s["n_nonfinite"] == 2
    assert abs(s["mean"] - 1.5) < 1e-15
    with pytest.raises(sl7.Sl7Error):
        sl7.stats_summary(np.zeros(14), _opts(4, 0.0, 4.0, 0.0))


def test_stats_quantile_outside_range_is_nan(lib):
    y = np.linspace(-1, 1, 1001)
    v = O.stats_vector(y, 0.0, -0.5, 0.5, 10)
    s = sl7.stats_summary(v, _opts(10, -0.5, 0.5, 0.0), q_levels=[0.1, 0.5, 0.9])
    assert math.isnan(s["quantiles"][0]) and math.isnan(s["quantiles"][2])
    assert abs(s["quantiles"][1]) <= 0.1


def test_product_package_never_imports_the_oracle():
    """The product path (paper_2302_05170_b200 and its C library) has no route to oracle/: importing the
    package and its modules in a fresh interpreter loads no oracle module, and no product source names it."""
    import subprocess
    import sys
    code = ("import sys, paper_2302_05170_b200, paper_2302_05170_b200.dist, paper_2302_05170_b200.build; "
            "print(any(m == 'oracle' or m.startswith('oracle.') for m in sys.modules))")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, cwd=ROOT, timeout=120)
    assert r.returncode == 0, r.stderr
    assert r.stdout.strip() == "False"
    pkg = os.path.join(ROOT, "paper_2302_05170_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                src = open(os.path.join(dirpath, f), encoding="utf-8", errors="replace").read()
                assert "import oracle" not in src and "from oracle" not in src and "sl7_oracle" not in src, f
