"""Oracle pins for the fission source and k (Alg. 1-2 P:341-417;
reading F1 in DESIGN.md): the analytic infinite-medium k_inf = nu Sigma_f / Sigma_a,
the exact two-point distribution of sites per absorption, the source resampling, power
iteration, and the degenerate cases."""
import math

import numpy as np
import pytest

import workloads

NUT = 0.55 / 0.25      # nu Sigma_f / Sigma_a = 2.2 for the infinite medium below


def _inf(oracle_mod):
    return oracle_mod.OracleModel.from_spec(workloads.infinite_medium(1.0, 0.25, 0.55))


def test_f1_sites_per_absorption_two_point(oracle_mod):
    """Infinite medium: every history ends in one absorption and banks floor(nut + xi) sites, i.e.
    2 or 3 with P(3) = frac(nut) = 0.2; the mean is nut = k_inf exactly in expectation."""
    m = _inf(oracle_mod)
    assert m.max_sites() == 3
    n = 20000
    res = m.run(n, seed=3, bank=True)
    c = res["counters"]
    assert c["absorptions"] == n and c["leaks"] == 0
    bn = res["bank_n"].astype(int)
    assert set(np.unique(bn).tolist()) <= {2, 3}
    p = NUT - math.floor(NUT)
    frac3 = (bn == 3).mean()
    assert abs(frac3 - p) < 4.5 * math.sqrt(p * (1 - p) / n)
    k = bn.sum() / n
    assert abs(k - NUT) < 4.5 * math.sqrt(p * (1 - p) / n)


def test_f1_sites_are_absorption_points(oracle_mod):
    """The banked sites of a history sit at its last collision point (trace), all equal."""
    m = _inf(oracle_mod)
    res = m.run(200, seed=4, bank=True, trace_cap=200000)
    tr = res["trace"]
    last = {}
    for rec in tr:
        last[int(rec["pid"])] = rec
    bank, bn = res["bank"], res["bank_n"]
    for h in range(200):
        assert last[h]["terminal"] == 1                         # absorbed
        sites = bank[h, :bn[h]]
        assert (sites == sites[0]).all()
        assert np.all(np.abs(sites[0]) <= 1.0)                  # inside the box


def test_f1_source_resampling(oracle_mod):
    """fission_source draws every source particle from the banked sites, uniformly: chi-square of
    the multiplicities of M sites over n_next draws, and isotropic unit directions."""
    m = _inf(oracle_mod)
    res = m.run(300, seed=5, bank=True)
    bank, bn = res["bank"], res["bank_n"]
    sites = np.concatenate([bank[h, :bn[h]] for h in range(300)])
    M = len(sites)
    n_next = 40 * M
    st, MM = m.fission_source(bank, bn, seed=5, cycle=0, n_next=n_next)
    assert MM == M
    pos = st[:3].T
    # map every drawn position to its site (positions of different histories differ)
    lookup = {tuple(s): i for i, s in enumerate(sites)}
    idx = np.array([lookup[tuple(p)] for p in pos])
    counts = np.bincount(idx, minlength=M)
    # sites of one history are identical points: aggregate per distinct position
    uniq, inv = np.unique(sites, axis=0, return_inverse=True)
    mult = np.bincount(inv, minlength=len(uniq))
    got = np.bincount(inv[idx], minlength=len(uniq))
    exp = n_next * mult / M
    chi2 = ((got - exp) ** 2 / exp).sum()
    dof = len(uniq) - 1
    assert chi2 < dof + 5 * math.sqrt(2 * dof)
    om = st[3:]
    assert np.allclose((om ** 2).sum(0), 1.0, atol=1e-14)
    assert abs(om[2].mean()) < 5 / math.sqrt(3 * n_next)


def test_f1_power_iteration_infinite_medium(oracle_mod):
    """Power iteration (Alg. 1): every cycle's k estimates k_inf = nu Sigma_f / Sigma_a."""
    m = _inf(oracle_mod)
    ks = m.power_iteration(4000, cycles=5, seed=7)
    p = NUT - math.floor(NUT)
    se = math.sqrt(p * (1 - p) / (4000 * 5))
    assert abs(np.mean(ks) - NUT) < 4.5 * se
    assert ks == m.power_iteration(4000, cycles=5, seed=7)          # deterministic


def test_f1_no_fission_collapses(oracle_mod):
    """nu Sigma_f = 0 everywhere: k = 0 and the next cycle has no source (error)."""
    m = oracle_mod.OracleModel.from_spec(workloads.infinite_medium(1.0, 0.25))
    res = m.run(100, seed=1, bank=True)
    assert res["bank_n"].sum() == 0
    with pytest.raises(RuntimeError, match="collapsed"):
        m.power_iteration(100, cycles=2)
