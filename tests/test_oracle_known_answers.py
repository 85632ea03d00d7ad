"""Pins the oracle (countmc_oracle.c) to the reference's own known-answer
tests, restated case by case (P: = /root/reference/proj/):
P:tests/test_rng.cpp, test_model.cpp, test_slice.cpp, test_streaming.cpp,
test_parallel.cpp.  CPU only."""
import math
from ctypes import POINTER, byref, c_double, c_uint64

import numpy as np
import pytest

import oracle
from oracle import load_oracle

ALL1 = 0xFFFFFFFFFFFFFFFF
L = load_oracle()


def philox(ctr, key):
    c = (c_uint64 * 4)(*ctr)
    k = (c_uint64 * 2)(*key)
    o = (c_uint64 * 4)()
    L.orc_philox4x64(c, k, o)
    return list(o)


# ------------------------------------------------------------ test_rng.cpp

@pytest.mark.parametrize("ctr,key,want", [
    ((0, 0, 0, 0), (0, 0),
     (0x16554d9eca36314c, 0xdb20fe9d672d0fdc, 0xd7e772cee186176b, 0x7e68b68aec7ba23b)),
    ((ALL1,) * 4, (ALL1, ALL1),
     (0x87b092c3013fe90b, 0x438c3c67be8d0224, 0x9cc7d7c69cd777b6, 0xa09caebf594f0ba0)),
    ((0x243f6a8885a308d3, 0x13198a2e03707344, 0xa4093822299f31d0, 0x082efa98ec4e6c89),
     (0x452821e638d01377, 0xbe5466cf34e90c6c),
     (0xa528f45403e61d95, 0x38c72dbd566e9788, 0xa5a1610e72fd18b5, 0x57bd43b5e52b7fe6)),
    ((2, 2, 3, 4), (5, 6),
     (0x92ab6a0e75619263, 0xd8ff75bdc6bf8f60, 0x450e124938725640, 0x94eb1a7cffd20cbb)),
])
def test_philox_known_answers(ctr, key, want):
    """P:tests/test_rng.cpp:19-56"""
    assert philox(ctr, key) == list(want)


def u01s(seed, chain, it, site, n):
    out = np.zeros(n)
    L.orc_stream_u01(seed, chain, it, site, n, out.ctypes.data_as(POINTER(c_double)))
    return out


def test_first_draw_addressing():
    """P:tests/test_rng.cpp:64-71: first draw comes from block (it, site, 0, 0)."""
    block = philox((5, 1234, 0, 0), (9, 2))
    want = ((block[0] >> 11) + 0.5) * 2.0 ** -53
    assert u01s(9, 2, 5, 1234, 1)[0] == want


def test_stream_determinism_and_open_interval():
    """P:tests/test_rng.cpp:58-62,82-94"""
    a = u01s(7, 3, 11, 42, 100)
    b = u01s(7, 3, 11, 42, 100)
    assert np.array_equal(a, b)
    x = u01s(1, 0, 0, 0, 100000)
    assert x.min() > 0.0 and x.max() < 1.0
    assert x.min() < 1e-3 and x.max() > 1 - 1e-3


def test_adjacent_sites_never_overlap():
    """P:tests/test_rng.cpp:73-80"""
    blocks = {tuple(philox((17, s, 0, 0), (1, 0))) for s in range(2000)}
    assert len(blocks) == 2000


def test_normal_quantile_values():
    """P:tests/test_rng.cpp:152-167"""
    q = L.orc_normal_quantile
    assert q(0.5) == 0.0
    assert q(0.975) == pytest.approx(1.9599639845400532, rel=1e-13)
    assert q(0.84) == pytest.approx(0.994457883209753, rel=1e-13)
    from statistics import NormalDist
    for p in (1e-10, 1e-4, 0.01, 0.2, 0.5, 0.7, 0.99, 1 - 1e-6):
        assert q(p) == pytest.approx(NormalDist().inv_cdf(p), rel=1e-9, abs=1e-12)
    for p in (0.01, 0.2, 0.3, 0.45):
        assert q(p) == pytest.approx(-q(1 - p), rel=1e-10)


# ---------------------------------------------------------- test_model.cpp

def test_epsilon_full_conditional_values():
    """P:tests/test_model.cpp:66-72"""
    f = L.orc_log_fc_epsilon
    assert f(0, 0.0, 0.0, 1.0, 0.0, None) == -1.0
    assert f(3, 0.5, -0.2, 2.0, 0.1, None) == pytest.approx(-1.1943246976412702, rel=1e-14)
    assert f(2, 0.0, 0.0, 0.5, -0.3, None) == pytest.approx(-1.430818220681718, rel=1e-14)


def test_gamma_fc_params():
    """P:tests/test_model.cpp:84-103"""
    sh, sc = c_double(), c_double()
    for nu, tau, eps, want in [(2.0, 1.0, [0.0, 0.0], (2.0, 1.0)),
                               (4.0, 2.0, [1.0, -1.0, 2.0], (3.5, 7.0)),
                               (1.0, 1.0, [0.5], (1.0, 0.625))]:
        e = np.array(eps)
        L.orc_gamma_fc_params(nu, tau, e.ctypes.data_as(POINTER(c_double)), len(eps),
                              byref(sh), byref(sc))
        assert (sh.value, sc.value) == want


def test_nu_full_conditional_values_and_support():
    """P:tests/test_model.cpp:123-131"""
    f = L.orc_log_fc_nu
    assert f(2.0, 1, 2.0, 0.0, 1.0, 1000.0) == pytest.approx(-1.3068528194400546, rel=1e-14)
    assert f(4.0, 2, 1.0, math.log(2.0), 1.5, 1000.0) == pytest.approx(-1.6137056388801096,
                                                                       rel=1e-14)
    for nu in (1001.0, 0.0, -2.0):
        assert f(nu, 1, 1.0, 0.0, 1.0, 1000.0) == -math.inf


def test_tau_theta_sigma_params():
    """P:tests/test_model.cpp:158-174,259-275,301-307"""
    sh, rt = c_double(), c_double()
    for args, want in [((1.0, 1.0, 2, 2.0, 1.5), (3.0, 2.5)), ((1.0, 1.0, 0, 2.0, 0.0), (1.0, 1.0)),
                       ((2.0, 3.0, 4, 1.0, 2.0), (4.0, 4.0))]:
        L.orc_tau_fc_params(*args, byref(sh), byref(rt))
        assert (sh.value, rt.value) == want
    mean, sd = c_double(), c_double()
    L.orc_theta_fc_params(0.0, 1, 1.0, 10.0, byref(mean), byref(sd))
    assert mean.value == 0.0 and sd.value == pytest.approx(0.9950371902099892, rel=1e-14)
    L.orc_theta_fc_params(0.0, 0, 1.0, 10.0, byref(mean), byref(sd))
    assert mean.value == 0.0 and sd.value == 10.0
    L.orc_theta_fc_params(5.0, 5, 1.0, 1e6, byref(mean), byref(sd))
    assert mean.value == pytest.approx(1.0, rel=1e-9) and sd.value == pytest.approx(math.sqrt(0.2), rel=1e-9)
    s = L.orc_log_fc_sigma
    assert s(1.0, 2, 0.0, 100.0) == 0.0
    assert s(0.5, 3, 1.2, 100.0) == pytest.approx(-0.32055845832016416, rel=1e-14)
    assert s(101.0, 3, 1.2, 100.0) == -math.inf and s(0.0, 3, 1.2, 100.0) == -math.inf


def test_clamped_exp_counts():
    """P:tests/test_model.cpp:309-317"""
    c = c_uint64(0)
    assert L.orc_clamped_exp(1.0, byref(c)) == math.exp(1.0) and c.value == 0
    assert L.orc_clamped_exp(900.0, byref(c)) == math.exp(700.0) and c.value == 1


# ---------------------------------------------------------- test_slice.cpp

class SliceCfg(__import__("ctypes").Structure):
    from ctypes import c_int, c_long
    _fields_ = [("max_step_out", c_int), ("burnin", c_long), ("tune_cutoff", c_long),
                ("w_init", c_double), ("max_shrink", c_int)]


def tune(w, wa, m, delta, cutoff):
    W, A = c_double(w), c_double(wa)
    cfg = SliceCfg(100, 0, cutoff, 1.0, 1000)
    L.orc_tune_update(byref(W), byref(A), m, delta, byref(cfg))
    return W.value, A.value


def test_tuning_constant_deltas_reproduce_step():
    """P:tests/test_slice.cpp:43-54"""
    for delta in (1.0, 0.37, 250.0):
        w, wa = 5.0, 0.0
        for m in range(1, 51):
            w, wa = tune(w, wa, m, delta, 0)
            assert w == pytest.approx(delta, rel=1e-12)
        assert w == delta


def test_tuning_zero_deltas_and_cutoff():
    """P:tests/test_slice.cpp:56-75"""
    w, wa = 2.5, 0.0
    for m in range(1, 21):
        w, wa = tune(w, wa, m, 0.0, 0)
    assert w == 2.5
    w, wa = 2.5, 0.0
    for m in range(1, 11):
        w, wa = tune(w, wa, m, 1.0, 10)
        assert w == 2.5
    assert wa == pytest.approx(55.0)
    w, wa = tune(w, wa, 11, 1.0, 10)
    assert w == pytest.approx(1.0, rel=1e-12)


def chain(density, x0, n, burnin, seed):
    out = np.zeros(n)
    rc = L.orc_slice_chain(density, x0, n, burnin, 1.0, seed, out.ctypes.data_as(POINTER(c_double)))
    assert rc == 0
    return out


def test_slice_bounded_support():
    """P:tests/test_slice.cpp:88-99"""
    x = chain(3, 0.5, 1000, 0, 3)
    assert np.all((x > 0) & (x < 1))


def ks(x, cdf):
    x = np.sort(x)
    n = len(x)
    F = np.array([cdf(v) for v in x])
    return max(np.max(np.arange(1, n + 1) / n - F), np.max(F - np.arange(n) / n))


def test_slice_chain_matches_standard_normal():
    """P:tests/test_slice.cpp:122-133 (KS at alpha = 0.01; 20k draws)"""
    from statistics import NormalDist
    x = chain(0, 0.0, 20000, 200, 12)
    assert abs(x.mean()) < 0.06 and 0.9 < x.var() < 1.1
    assert ks(x[::5], NormalDist().cdf) < 1.63 / math.sqrt(len(x[::5]))


def test_slice_chain_matches_gamma_and_invgamma():
    """P:tests/test_slice.cpp:135-161"""
    g = chain(1, 1.0, 20000, 200, 21)
    assert g.mean() == pytest.approx(1.5, rel=0.05)       # Gamma(3, rate 2)
    ig = chain(2, 1.0, 20000, 200, 33)
    assert (1 / ig).mean() == pytest.approx(2 / 3, rel=0.05)  # 1/x ~ Gamma(2, rate 3)


# ------------------------------------------ test_streaming / test_parallel

def moments(v):
    m, ms = c_double(), c_double()
    a = np.ascontiguousarray(v, dtype=np.float64)
    L.orc_moments_stream(a.ctypes.data_as(POINTER(c_double)), len(a), byref(m), byref(ms))
    return m.value, ms.value


def test_moments_hand_cases():
    """P:tests/test_streaming.cpp:16-31"""
    m, ms = moments([3.25] * 7)
    assert m == 3.25 and ms == pytest.approx(3.25 ** 2, rel=1e-15)
    m, ms = moments([1.0, 2.0, 3.0])
    assert m == pytest.approx(2.0, rel=1e-15) and ms == pytest.approx(14 / 3, rel=1e-15)


def test_moments_two_pass_and_offset_stress():
    """P:tests/test_streaming.cpp:33-60 (offset stream shortened to 2e5)"""
    rng = np.random.default_rng(31415)
    v = rng.normal(2.0, 5.0, 10000)
    m, ms = moments(v)
    assert m == pytest.approx(math.fsum(v) / len(v), rel=1e-12)
    assert ms == pytest.approx(math.fsum(v * v) / len(v), rel=1e-12)
    v = 1e9 + np.random.default_rng(99).uniform(0, 1, 200000)
    m, _ = moments(v)
    assert abs(m - math.fsum(v) / len(v)) < 1e-6


def test_pairwise_and_det_sum():
    """P:tests/test_parallel.cpp:46-85"""
    rng = np.random.default_rng(5)
    x = (rng.uniform(size=12345) - 0.5) * 1e6
    p = x.ctypes.data_as(POINTER(c_double))
    assert L.orc_pairwise_sum(p, len(x)) == pytest.approx(math.fsum(x), rel=1e-12)
    assert L.orc_pairwise_sum(p, 0) == 0.0 and L.orc_pairwise_sum(p, 1) == x[0]
    y = np.cos(0.01 * np.arange(54321)) * 1e3
    assert L.orc_det_sum(y.ctypes.data_as(POINTER(c_double)), len(y)) == \
        pytest.approx(math.fsum(y), rel=1e-12)


def test_disjunction_combine():
    """P:tests/test_streaming.cpp:215-222"""
    d = L.orc_disjunction_combine
    assert d(0.3, 0.4, 0.1) == pytest.approx(0.6, rel=1e-15)
    for p in (0.0, 0.25, 1.0):
        assert d(p, p, p) == pytest.approx(p, rel=1e-15)
    assert d(1.0, 0.0, 0.0) == 1.0 and d(0.9, 0.9, 0.5) == 1.0 and d(0.0, 0.0, 0.1) == 0.0
