"""Oracle pins P1/P2 and the spec'd transcendentals (reading R-T) against things
other than the oracle itself: published Philox KAT vectors, closed forms, libm."""
import math
import os

import numpy as np
import pytest

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _rows(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return [ln.split() for ln in f if ln.strip() and not ln.startswith("#")]


def test_philox_kat(oracle_mod):
    """P1: Random123 Philox4x32-10 known-answer vectors (tests/golden/philox4x32_10_kat.txt)."""
    rows = _rows("philox4x32_10_kat.txt")
    assert len(rows) == 3
    for r in rows:
        v = [int(x, 16) for x in r]
        out = oracle_mod.philox(v[0:4], v[4:6])
        assert [int(x) for x in out] == v[6:10]


def test_u01_exact_range(oracle_mod):
    """P2: U(h,l) = ((((h<<32)|l)>>12)+0.5) 2^-52 is exact, in (0,1), endpoints 2^-53 / 1-2^-53."""
    assert oracle_mod.u01(0, 0) == 2.0 ** -53
    assert oracle_mod.u01(0xFFFFFFFF, 0xFFFFFFFF) == 1.0 - 2.0 ** -53
    rng = np.random.default_rng(0)
    for h, l in rng.integers(0, 2 ** 32, size=(200, 2)):
        k = ((int(h) << 32) | int(l)) >> 12
        assert oracle_mod.u01(int(h), int(l)) == (k + 0.5) / 2.0 ** 52   # exact closed form
        assert 0.0 < oracle_mod.u01(int(h), int(l)) < 1.0


def _ulp_err(a, b):
    return abs(a - b) / math.ulp(b) if b != 0 else abs(a)


def test_log_against_libm(oracle_mod):
    """R-T: the spec'd log agrees with libm's correctly-rounded-ish log to <= 2 ulp."""
    rng = np.random.default_rng(1)
    xs = list(rng.random(20000)) + [2.0 ** -53, 1.0 - 2.0 ** -53, 0.5, 0.25, 0.7071067811865476,
                                    0.7071067811865475, 0.999999, 1e-10, 0.1, 0.9]
    xs += list(2.0 ** -rng.uniform(0, 53, 5000))
    worst = 0.0
    for x in xs:
        x = float(x)
        if x <= 0.0:
            continue
        worst = max(worst, _ulp_err(oracle_mod.log(x), math.log(x)))
    assert worst <= 2.0, worst
    assert oracle_mod.log(0.5) == -math.log(2.0)
    assert oracle_mod.log(1.0) == 0.0


def test_sincos2pi_against_libm(oracle_mod):
    """R-T: cos/sin(2 pi xi) within 2e-16 absolute of libm, c^2+s^2 = 1, exact quadrant points."""
    rng = np.random.default_rng(2)
    worst = 0.0
    for xi in rng.random(20000):
        xi = float(xi)
        c, s = oracle_mod.sincos2pi(xi)
        # libm reference evaluated on the exact-quadrant reduced argument to avoid the
        # rounding of 2*pi*xi itself: cos(2 pi xi) = cos(pi/2 * (4 xi)) with 4 xi exact
        x4 = xi * 4.0
        q = math.floor(x4)
        f = x4 - q
        cf, sf = math.cos(f * math.pi / 2), math.sin(f * math.pi / 2)
        ref = [(cf, sf), (-sf, cf), (-cf, -sf), (sf, -cf)][q]
        worst = max(worst, abs(c - ref[0]), abs(s - ref[1]))
        assert abs(c * c + s * s - 1.0) < 1e-15
    assert worst < 3e-16, worst
    c, s = oracle_mod.sincos2pi(0.25)
    assert abs(c) == 0.0 and s == 1.0
    c, s = oracle_mod.sincos2pi(0.5)
    assert c == -1.0 and abs(s) == 0.0
    c, s = oracle_mod.sincos2pi(0.125)
    assert abs(c - math.sqrt(0.5)) <= 1.2e-16 and abs(s - math.sqrt(0.5)) <= 1.2e-16


def test_exponential_mean(oracle_mod):
    """tau = -ln xi over the Philox stream has mean 1 and variance 1 (Exp(1))."""
    taus = []
    for pid in range(40000):
        o = oracle_mod.philox([pid, 0, 0, 0], [1, 0])
        taus.append(-oracle_mod.log(oracle_mod.u01(int(o[2]), int(o[3]))))
    taus = np.array(taus)
    n = len(taus)
    assert abs(taus.mean() - 1.0) < 4.0 / math.sqrt(n)
    assert abs(taus.var() - 1.0) < 4.0 * math.sqrt(8.0 / n)


def _iso_draws(oracle_mod, n, seed=17):
    """(xi_mu, xi_phi) of epoch-0 block 1 (O17) for pids 0..n-1."""
    key = [seed & 0xFFFFFFFF, seed >> 32]
    out = np.zeros((n, 2))
    for pid in range(n):
        x = oracle_mod.philox([pid, 0, 0, 1], key)
        out[pid] = (oracle_mod.u01(int(x[0]), int(x[1])), oracle_mod.u01(int(x[2]), int(x[3])))
    return out


def test_iso_worked_values(oracle_mod):
    """O15 closed forms: mu = 2 xi_mu - 1, phi = 2 pi xi_phi, Omega = (s cos phi, s sin phi, mu),
    s = sqrt(1 - mu^2).  A phi = pi xi (or a swapped sin / cos, or a dropped s) fails these."""
    h = math.sqrt(0.75)
    cases = [((0.5, 0.0), (1.0, 0.0, 0.0)),
             ((0.5, 0.25), (0.0, 1.0, 0.0)),
             ((0.5, 0.5), (-1.0, 0.0, 0.0)),
             ((0.5, 0.75), (0.0, -1.0, 0.0)),
             ((0.75, 0.125), (h / math.sqrt(2.0), h / math.sqrt(2.0), 0.5)),
             ((0.25, 0.625), (-h / math.sqrt(2.0), -h / math.sqrt(2.0), -0.5)),
             ((0.75, 1.0 / 6.0), (h * 0.5, h * h, 0.5)),
             ((1.0, 0.3), (0.0, 0.0, 1.0))]
    for (xm, xp), want in cases:
        got = oracle_mod.iso(xm, xp)
        assert np.allclose(got, want, rtol=0, atol=4e-16), ((xm, xp), got, want)


def test_iso_statistics(oracle_mod):
    """O15 pins on Philox-drawn directions: |Omega| = 1, E[Omega] = 0 and E[Omega_i^2] = 1/3
    (4 sigma; Var Omega_i = 1/3, Var Omega_i^2 = 1/5 - 1/9 = 4/45 on the unit sphere), and
    Kolmogorov-Smirnov: mu = Omega_z ~ U(-1, 1), azimuth atan2(Omega_y, Omega_x) ~ U(-pi, pi),
    and the azimuth in every octant-pair of mu is uniform too (no mu-phi coupling)."""
    from scipy import stats
    n = 20000
    xi = _iso_draws(oracle_mod, n)
    om = np.array([oracle_mod.iso(a, b) for a, b in xi])
    assert np.all(np.abs(np.linalg.norm(om, axis=1) - 1.0) <= 4e-16)
    mean = om.mean(axis=0)
    assert np.all(np.abs(mean) <= 4.0 * math.sqrt(1.0 / 3.0 / n)), mean
    sq = (om ** 2).mean(axis=0)
    assert np.all(np.abs(sq - 1.0 / 3.0) <= 4.0 * math.sqrt(4.0 / 45.0 / n)), sq
    assert stats.kstest(om[:, 2], stats.uniform(loc=-1.0, scale=2.0).cdf).pvalue > 1e-3
    phi = np.arctan2(om[:, 1], om[:, 0])
    assert stats.kstest(phi, stats.uniform(loc=-math.pi, scale=2.0 * math.pi).cdf).pvalue > 1e-3
    for lo, hi in ((-1.0, -0.5), (-0.5, 0.0), (0.0, 0.5), (0.5, 1.0)):
        sel = (om[:, 2] >= lo) & (om[:, 2] < hi)
        assert stats.kstest(phi[sel], stats.uniform(loc=-math.pi, scale=2.0 * math.pi).cdf).pvalue > 1e-4
