"""CPU-only checks of the host side: the C ABI library loads and exports every
entry point include/fsmc.h declares, the device math compiles as host C++ and
reproduces glibc/scipy bit for bit, and the pure-host API (machine shapes,
key splitting, cost model, argument validation) behaves like the reference."""

import ctypes
import math
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2503_17405_b200", "libfsmc.so")
HDR = os.path.join(ROOT, "include", "fsmc.h")


def declared_symbols():
    text = open(HDR).read()
    return sorted(set(re.findall(r"\b(fsmc_[a-z_]+)\s*\(", text)))


def test_library_exports_every_declared_entry_point():
    if not os.path.exists(LIB):
        pytest.skip("libfsmc.so not built")
    lib = ctypes.CDLL(LIB)
    syms = declared_symbols()
    assert "fsmc_run" in syms and "fsmc_init" in syms and "fsmc_lockstep_run" in syms
    for s in syms:
        assert hasattr(lib, s), s
    lib.fsmc_abi_version.restype = ctypes.c_int32
    hdr = open(os.path.join(ROOT, "include", "fsmc.h")).read()
    abi = int(re.search(r"#define FSMC_ABI_VERSION (\d+)", hdr).group(1))
    assert lib.fsmc_abi_version() == abi   # fsmc.h FSMC_ABI_VERSION


def test_state_without_work_words_is_rejected_before_any_launch():
    """Launch bookkeeping (chain queues, barrier words) lives in each state
    block's own work[] words, so concurrent runs on different batches never
    share it; a state without them is an argument error (no CUDA call made)."""
    if not os.path.exists(LIB):
        pytest.skip("libfsmc.so not built")
    from paper_2503_17405_b200 import _lib as L
    lib = ctypes.CDLL(LIB)
    lib.fsmc_last_error.restype = ctypes.c_char_p
    k = L.Kernel()
    k.family, k.max_tries, k.proposal_scale = L.DRMH, 10, 0.1
    t = L.Target()
    t.kind, t.dim = 8, 2   # FSMC_T_FLAT
    st = L.State()
    st.m, st.dim, st.n_vec, st.n_scal = 4, 2, 2, 3
    st.vec = st.scal = st.ints = st.err_key = 16   # never dereferenced: rejected first
    st.work = None
    out = L.Outputs()
    rc = lib.fsmc_run(ctypes.byref(k), ctypes.byref(t), ctypes.byref(st), ctypes.c_int64(10), 0,
                      None, ctypes.c_int64(1 << 40), 0, ctypes.byref(out), 0, None)
    assert rc == 1 and b"work" in lib.fsmc_last_error()


def test_library_is_sm100a():
    if not os.path.exists(LIB):
        pytest.skip("libfsmc.so not built")
    out = subprocess.run(["cuobjdump", "--list-elf", LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out


HOST_HARNESS = r"""
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include "dmath.cuh"
#include "prng.cuh"
extern "C" double h_log(double x) { return fsmc::gl_log(x); }
extern "C" double h_ndtri(double x) { return fsmc::ndtri(x); }
extern "C" double h_softplus(double a) { return fsmc::softplus_neg(a); }
extern "C" double h_exp(double x) { return fsmc::gl_exp(x); }
extern "C" long h_exp_mismatch(long n, unsigned long long s) {
  long bad = 0;
  for (long t = 0; t < n; t++) {
    s ^= s << 13; s ^= s >> 7; s ^= s << 17;
    const double v = (s >> 11) * 0x1p-53;
    double x;
    switch (t % 6) {
      case 0: x = -v * 750.0; break;                    // accept tests, MoG modes
      case 1: x = -708.0 - v * 40.0; break;             // subnormal results (special case)
      case 2: x = v * 712.0; break;                     // overflow side
      case 3: x = (v - 0.5) * 1e-15; break;             // tiny |x|
      case 4: x = -745.1332191019411 - v * 0.1; break;  // underflow boundary
      default: { unsigned long long u = s; std::memcpy(&x, &u, 8); }
    }
    double a = std::exp(x), b = fsmc::gl_exp(x);
    if (std::memcmp(&a, &b, 8) != 0 && !(std::isnan(a) && std::isnan(b))) bad++;
  }
  return bad;
}
extern "C" double h_normal(unsigned long long seed, unsigned long long stream,
                           unsigned long long ctr) {
  return fsmc::normal(fsmc::hash_seed_stream(seed, stream), ctr);
}
extern "C" long h_log_mismatch(long n, unsigned long long s) {
  long bad = 0;
  for (long t = 0; t < n; t++) {
    s ^= s << 13; s ^= s >> 7; s ^= s << 17;
    double x;
    switch (t & 3) {
      case 0: x = ((s >> 11) + 0.5) * 0x1p-53 * 0.1353352832366127; break;  // ndtri tail args
      case 1: x = 2.0 + ((s >> 11) * 0x1p-53) * 7.0; break;                 // sqrt(-2 log y)
      case 2: x = 1.0 - (s >> 11) * 0x1p-53; break;                          // 1 - u
      default: { unsigned long long u = s & 0x7fefffffffffffffULL; std::memcpy(&x, &u, 8); }
    }
    double a = std::log(x), b = fsmc::gl_log(x);
    if (std::memcmp(&a, &b, 8) != 0) bad++;
  }
  return bad;
}
"""


@pytest.fixture(scope="module")
def host_math(tmp_path_factory):
    d = tmp_path_factory.mktemp("hostmath")
    src = d / "h.cpp"
    src.write_text(HOST_HARNESS)
    so = d / "libh.so"
    csrc = os.path.join(ROOT, "paper_2503_17405_b200", "csrc")
    subprocess.check_call(["g++", "-O2", "-ffp-contract=off", "-mfma", "-std=c++17", "-fPIC",
                           "-shared", f"-I{csrc}", "-o", str(so), str(src)])
    h = ctypes.CDLL(str(so))
    for f in ("h_log", "h_ndtri", "h_softplus", "h_exp"):
        getattr(h, f).restype = ctypes.c_double
        getattr(h, f).argtypes = [ctypes.c_double]
    h.h_normal.restype = ctypes.c_double
    h.h_normal.argtypes = [ctypes.c_ulonglong] * 3
    h.h_log_mismatch.restype = ctypes.c_long
    h.h_log_mismatch.argtypes = [ctypes.c_long, ctypes.c_ulonglong]
    h.h_exp_mismatch.restype = ctypes.c_long
    h.h_exp_mismatch.argtypes = [ctypes.c_long, ctypes.c_ulonglong]
    return h


def test_branch_free_softplus_is_accurate(host_math):
    """softplus_neg(a) = log1p(exp(-a)) (logistic likelihood, NUTS logaddexp)
    within 2 ulp of the correctly rounded value over [0, 745] and at the
    range ends."""
    from fractions import Fraction  # noqa: F401  (exactness reference below is mpmath)
    mpmath = pytest.importorskip("mpmath")
    mpmath.mp.prec = 200
    rng = np.random.default_rng(7)
    a = np.concatenate([rng.uniform(0, 1, 3000), rng.uniform(0, 40, 3000),
                        rng.exponential(3.0, 2000), rng.uniform(40, 745, 500),
                        [0.0, 1e-300, 5e-324, 1e-17, 0.34657359027997264, 0.6931471805599453,
                         1.0, 36.7, 37.5, 700.0, 709.0, 745.0]])
    worst = 0.0
    for v in a:
        got = host_math.h_softplus(float(v))
        ref = float(mpmath.log1p(mpmath.exp(-mpmath.mpf(float(v)))))
        if v > 700:      # clamped at e^-700: the term is below any sum's resolution
            assert 0.0 <= got <= 1e-303
            continue
        ulp = math.ulp(ref)
        worst = max(worst, abs(got - ref) / ulp)
    assert worst <= 2.0, worst


def test_glibc_log_restatement_is_bit_exact(host_math):
    assert host_math.h_log_mismatch(2_000_000, 88172645463325252) == 0
    for x in (1.0, 0.5, 2.0, 1e-300, 5e-324, 0.9999999999, 1.0625):
        assert host_math.h_log(x) == math.log(x)


def test_glibc_exp_restatement_is_bit_exact(host_math):
    """gl_exp (dmath.cuh) is Python's math.exp bit for bit: the DRMH accept test
    (drmh.py:58-59) and the NUTS exponentials (nuts.py:45, 172, 201)."""
    assert host_math.h_exp_mismatch(3_000_000, 0x9E3779B97F4A7C15) == 0
    for x in (0.0, -0.0, 1e-300, -1e-17, 1.0, -1.0, 709.782712893384, 709.7827128933841,
              -708.3964185322641, -745.1332191019411, -745.1332191019412, -1e4, 1e4,
              float("inf"), float("-inf")):
        try:
            ref = math.exp(x)
        except OverflowError:   # Python raises where libm returns +inf
            ref = math.inf
        assert host_math.h_exp(x) == ref, x


def test_ndtri_restatement_matches_scipy(host_math):
    from scipy.special import ndtri
    rng = np.random.default_rng(3)
    b = rng.integers(0, 2**53, size=50_000, dtype=np.int64)
    y = (b.astype(np.float64) + 0.5) * 2.0**-53
    ref = ndtri(y)
    got = np.array([host_math.h_ndtri(v) for v in y])
    assert np.array_equal(got, ref)
    edge = np.array([0.5 * 2.0**-53, 1e-20, 0.13533528323661269189, 0.8646647167633873,
                     0.86466471676338730811, 1 - 2.0**-53])
    assert np.array_equal(np.array([host_math.h_ndtri(v) for v in edge]), ndtri(edge))


def test_device_prng_matches_golden_known_answers(host_math):
    from golden_cases import load
    p = load("prng")
    for t, z in zip(p["trip"], p["normal"]):
        assert host_math.h_normal(*[int(v) for v in t]) == z


# ---------------------------------------------------------------- host API
def test_split_and_keys_match_reference_goldens():
    from golden_cases import load
    from paper_2503_17405_b200 import prng
    p = load("prng")
    kids = prng.split(prng.key(0), 3) + prng.split(prng.key(7, 99), 5)
    assert [k.stream for k in kids] == [int(s) for s in p["split_streams"]]
    k = prng.key(2**70 + 5, stream=2**64, counter=-1 & (2**64 - 1))
    assert k.seed == (2**70 + 5) & (2**64 - 1) and k.stream == 0
    with pytest.raises(ValueError):
        prng.split(prng.key(0), 0)
    assert prng.split(prng.key(5, 11), 8)[:3] == prng.split(prng.key(5, 11), 3)


def test_machine_shapes_and_bundled_orders():
    from paper_2503_17405_b200 import fsm
    import paper_2503_17405_b200 as fm
    d = fm.drmh_kernel(10, 0.5)
    assert d.fsm.labels == ("INIT", "PROPOSE", "DONE") and (2, 2) in d.fsm.edges
    n = fm.nuts_kernel(0.1, 5)
    assert n.fsm.labels == ("INIT", "DOUBLE", "INTEGRATE", "CHECK", "DONE")
    assert fsm.default_bundled_order(n.fsm) == (5, 1, 2, 3, 4)
    fsm.validate_bundled_order(d.fsm, (3, 2, 1))
    with pytest.raises(fsm.FsmError):
        fsm.validate_bundled_order(d.fsm, (1, 2, 3))
    with pytest.raises(fsm.FsmError):
        fsm.FsmDefinition(labels=("A", "B"), edges=frozenset({(1, 2), (2, 2)}))
    assert "doublecircle" in fsm.topology_as_graphviz(d.fsm)
    assert fsm.topology_as_dict(n.fsm)["loop_states"] == [2, 3, 4]
    e = fm.elliptical_kernel()
    assert e.default_costs.shared_sites == (1, 1, 0)


def test_kernel_argument_validation():
    import paper_2503_17405_b200 as fm
    with pytest.raises(fm.KernelError):
        fm.drmh_kernel(0, 1.0)
    with pytest.raises(fm.KernelError):
        fm.drmh_kernel(3, 0.0)
    with pytest.raises(fm.KernelError):
        fm.nuts_kernel(0.0)
    with pytest.raises(fm.KernelError):
        fm.nuts_kernel(0.1, max_depth=0)
    with pytest.raises(fm.KernelError):
        fm.elliptical_kernel().check_target(fm.standard_normal_target(2))


def test_cost_model_matches_reference_semantics():
    import paper_2503_17405_b200 as fm
    from paper_2503_17405_b200.lockstep import CostParams
    e = fm.elliptical_kernel()
    c = e.default_costs
    assert c.tick_cost("plain") == pytest.approx(0.02 + 1.0 + 0.02 + 1.0 + 0.01)
    assert c.tick_cost("amortized") == pytest.approx(0.05 + 1.0)
    assert c.shared_evals_per_tick("plain") == 2 and c.shared_evals_per_tick("amortized") == 1
    with pytest.raises(ValueError):
        CostParams(block_costs=(1.0, 1.0), alpha=0.1)


def test_target_constants_follow_the_reference():
    import paper_2503_17405_b200 as fm
    from paper_2503_17405_b200 import _lib
    t = fm.correlated_mog_target(10, 0.9, [-3.0, 0.0, 3.0])
    L = np.linalg.cholesky(fm.equicorrelated_covariance(10, 0.9))
    assert t.log_norm == -0.5 * 10 * math.log(2 * math.pi) - float(np.sum(np.log(np.diag(L)))) - math.log(3)
    assert t.kind == _lib.T_MOG and t.a == pytest.approx(10.0) and t.b == pytest.approx(1 / 9.1)
    g = fm.gaussian_target(np.zeros(100), np.linalg.cholesky(fm.equicorrelated_covariance(100, 0.99)))
    assert g.kind == _lib.T_GAUSS_EQUICORR
    g = fm.gaussian_target(np.zeros(3), np.array([[1.0, 0, 0], [0.3, 0.8, 0], [-0.2, 0.1, 0.5]]))
    assert g.kind == _lib.T_GAUSS_DENSE
    assert fm.conjugate_target(5).gaussian_prior is not None
    with pytest.raises(fm.TargetError):
        fm.gaussian_target(np.zeros(2), np.array([[1.0, 0.5], [0.0, 1.0]]))
