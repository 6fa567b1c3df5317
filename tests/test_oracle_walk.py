"""Oracle walk pins: P8 chord, P9 volume recovery, P10 infinite medium,
P11 particle balance, P12 nested == flat, P14 additivity, P17 closedness, and the exact
counter invariants of the walk (§8(c)2)."""
import math
import os

import numpy as np
import pytest

import workloads

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
CFGS = ["c1", "c2", "c3", "c4", "c5m", "c5r"]


def _invariants(c):
    assert c["segments"] == c["crossings"] + c["reflections"] + c["collisions"]
    assert c["particles"] == c["absorptions"] + c["leaks"] + c["lost"] + c["capped"]
    assert c["crossings"] == c["leaks"] + sum(c[f"cross_l{i}"] for i in range(8))


@pytest.mark.parametrize("cfg", CFGS)
def test_p17_closed_and_invariants(oracle_mod, cfg):
    """P17: every walk terminates, LOST = CAPPED = 0; counter identities hold exactly."""
    spec, _ = workloads.config(cfg)
    m = oracle_mod.OracleModel.from_spec(spec)
    res = m.run(400, seed=3, pflags=True)
    c = res["counters"]
    _invariants(c)
    assert c["particles"] == 400 and c["lost"] == 0 and c["capped"] == 0
    assert c["flagged"] == int((res["pflags"] != 0).sum())
    assert res["exits"].sum() == c["crossings"]
    assert (res["len"] >= 0).all() and res["len"].sum() > 0


def test_trace_matches_tallies(oracle_mod):
    """The per-segment trace sums to the per-cell tallies (same walk, two outputs)."""
    spec, _ = workloads.config("c2")
    m = oracle_mod.OracleModel.from_spec(spec)
    res = m.run(300, seed=1, trace_cap=200000)
    tr = res["trace"]
    seg = tr[tr["level"] != -1]
    seg = tr[(tr["terminal"] != 3) | (tr["s"] > 0)]
    cell_to_mc = {int(c): i for i, c in enumerate(m.mc_cell)}
    acc = np.zeros(m.n_mc)
    for rec in seg:
        if rec["cell_before"] >= 0:
            acc[cell_to_mc[int(rec["cell_before"])]] += rec["s"]
    assert np.allclose(acc, res["len"], rtol=1e-12, atol=0)
    assert len(tr) == res["counters"]["segments"]


def test_p8_chord_single_ray(oracle_mod):
    """P8: deterministic ray through the void pincell (tests/golden/chord_c1_void.txt)."""
    spec = workloads.c1_pincell(bc="vacuum", void=True)
    m = oracle_mod.OracleModel.from_spec(spec)
    st = np.array([[0.0], [0.0], [100.0], [1.0], [0.0], [0.0]])
    res = m.run(1, states=st, trace_cap=16)
    with open(os.path.join(GOLDEN, "chord_c1_void.txt")) as f:
        rows = [ln.split() for ln in f if ln.strip() and not ln.startswith("#")]
    exp = [float(r[1]) for r in rows]
    got = res["trace"]["s"]
    assert len(got) == 4
    assert np.allclose(got, exp, rtol=1e-12, atol=1e-15)
    assert abs(got.sum() - 0.63) < 1e-15


def test_p8_chord_invariant(oracle_mod):
    """P8: all-void model, VACUUM box: sum of segment lengths = slab exit distance."""
    spec = workloads.c1_pincell(bc="vacuum", void=True)
    m = oracle_mod.OracleModel.from_spec(spec)
    n = 3000
    rng = np.random.default_rng(11)
    lo = np.array(spec["source"]["lo"])
    hi = np.array(spec["source"]["hi"])
    r = rng.uniform(lo, hi, size=(n, 3))
    om = rng.normal(size=(n, 3))
    om /= np.linalg.norm(om, axis=1, keepdims=True)
    st = np.concatenate([r.T, om.T])
    res = m.run(n, states=st, trace_cap=200000)
    tr = res["trace"]
    c = res["counters"]
    assert c["segments"] == c["crossings"] and c["leaks"] == n and c["collisions"] == 0
    sums = np.zeros(n)
    np.add.at(sums, tr["pid"].astype(np.int64), tr["s"])
    with np.errstate(divide="ignore"):
        ex = np.where(om > 0, (hi - r) / om, np.where(om < 0, (lo - r) / om, np.inf)).min(axis=1)
    assert np.allclose(sums, ex, rtol=1e-12, atol=1e-13)


def test_p9_volume_recovery(oracle_mod):
    """P9: uniform Sigma everywhere + all-REFLECT box => E[L_c]/E[L_tot] = V_c / V_box."""
    spec = workloads.c1_pincell(uniform=(1.0, 0.1))
    m = oracle_mod.OracleModel.from_spec(spec)
    p = workloads.models.PIN_PITCH
    r = workloads.models.PIN_R
    area = [math.pi * r[0] ** 2, math.pi * (r[1] ** 2 - r[0] ** 2), math.pi * (r[2] ** 2 - r[1] ** 2)]
    area.append(p * p - sum(area))
    exact = np.array(area) / (p * p)
    B, nb = 20, 1500
    fr = []
    for b in range(B):
        res = m.run(nb, seed=7, pid_begin=b * nb)
        fr.append(res["len"] / res["len"].sum())
    fr = np.array(fr)
    mean, se = fr.mean(0), fr.std(0, ddof=1) / math.sqrt(B)
    assert (np.abs(mean - exact) < 4.5 * se + 1e-4).all(), (mean, exact, se)


def test_p10_infinite_medium(oracle_mod):
    """P10: one material, REFLECT box, Sigma_t=1, Sigma_a=0.25: track length per history
    ~ Exp(Sigma_a) (mean 4, var 16); collisions ~ Geom(1/4) (mean 4, var 12)."""
    from scipy import stats
    spec = workloads.infinite_medium(1.0, 0.25)
    m = oracle_mod.OracleModel.from_spec(spec)
    n = 4000
    res = m.run(n, seed=5, trace_cap=400000)
    c = res["counters"]
    assert c["absorptions"] == n and c["leaks"] == 0
    tr = res["trace"]
    L = np.zeros(n)
    np.add.at(L, tr["pid"].astype(np.int64), tr["s"])
    K = np.zeros(n)
    np.add.at(K, tr["pid"].astype(np.int64), (tr["kind"] == 3).astype(float))
    assert abs(L.mean() - 4.0) < 4 * 4.0 / math.sqrt(n)
    assert abs(K.mean() - 4.0) < 4 * math.sqrt(12.0 / n)
    assert abs(K.var() - 12.0) < 2.5
    assert stats.kstest(L, "expon", args=(0, 4.0)).pvalue > 1e-3
    assert abs(res["len"].sum() / n - 4.0) < 4 * 4.0 / math.sqrt(n)


@pytest.mark.parametrize("cfg", ["c1", "c2"])
def test_p11_particle_balance(oracle_mod, cfg):
    """P11: in a reflective model every history ends in absorption, and the track-length
    estimate of absorptions sum_c Sigma_a(c) len_c / N -> 1."""
    spec, _ = workloads.config(cfg)
    m = oracle_mod.OracleModel.from_spec(spec)
    sa = np.array([spec["materials"][m.cell_material(int(c))]["sigma_a"] for c in m.mc_cell])
    B, nb = 10, 600
    est = []
    for b in range(B):
        res = m.run(nb, seed=9, pid_begin=b * nb)
        assert res["counters"]["absorptions"] == nb
        est.append((sa * res["len"]).sum() / nb)
    est = np.array(est)
    assert abs(est.mean() - 1.0) < 4.5 * est.std(ddof=1) / math.sqrt(B) + 2e-3


def test_p12_nested_equals_flat(oracle_mod):
    """P12: 3x3 lattice nested (root -> RECT -> pin) vs the same geometry as one flat CSG
    universe: identical event/material sequences and bit-identical segment lengths."""
    a = oracle_mod.OracleModel.from_spec(workloads.lattice3_nested(flat=False))
    b = oracle_mod.OracleModel.from_spec(workloads.lattice3_nested(flat=True))
    n = 400
    ra = a.run(n, seed=2, trace_cap=200000)
    rb = b.run(n, seed=2, trace_cap=200000)
    ta, tb = ra["trace"], rb["trace"]
    assert len(ta) == len(tb)
    assert np.array_equal(ta["pid"], tb["pid"]) and np.array_equal(ta["kind"], tb["kind"])
    ma = np.array([a.cell_material(int(c)) for c in ta["cell_before"]])
    mb = np.array([b.cell_material(int(c)) for c in tb["cell_before"]])
    assert np.array_equal(ma, mb)
    assert np.array_equal(ta["s"], tb["s"])


def test_p14_additivity_and_determinism(oracle_mod):
    """P14: out(A u B) = out(A) + out(B): counters exact, lengths to summation order."""
    spec, _ = workloads.config("c2")
    m = oracle_mod.OracleModel.from_spec(spec)
    ab = m.run(600, seed=4, pid_begin=1000)
    a = m.run(250, seed=4, pid_begin=1000)
    b = m.run(350, seed=4, pid_begin=1250)
    assert ab["counters"] == {k: a["counters"][k] + b["counters"][k] for k in ab["counters"]}
    assert np.array_equal(ab["exits"], a["exits"] + b["exits"])
    assert np.allclose(ab["len"], a["len"] + b["len"], rtol=1e-13, atol=0)
    again = m.run(600, seed=4, pid_begin=1000)
    assert np.array_equal(again["out"], ab["out"])
    one = m.run(600, seed=4, pid_begin=1000, threads=1)
    assert one["counters"] == ab["counters"]
    assert np.allclose(one["len"], ab["len"], rtol=1e-13, atol=0)


def test_o13_exact_coincidence_resolves_to_top(oracle_mod):
    """O13: C5's root box coincides exactly with the top lattice's outer walls; the tie goes
    to the root (a reflection, level 0) and is not flagged."""
    spec, _ = workloads.config("c5r")
    m = oracle_mod.OracleModel.from_spec(spec)
    res = m.run(300, seed=1, pflags=True)
    c = res["counters"]
    assert c["reflections"] > 0 and c["lost"] == 0 and c["flagged"] == 0


def test_seed_changes_walks(oracle_mod):
    spec, _ = workloads.config("c1")
    m = oracle_mod.OracleModel.from_spec(spec)
    a = m.run(200, seed=1)
    b = m.run(200, seed=2)
    assert a["counters"]["segments"] != b["counters"]["segments"]


@pytest.mark.parametrize("cfg", ["c1", "c3", "c4"])
def test_per_history_outputs_match_trace(oracle_mod, cfg):
    """The oracle's per-history segment count and terminal equal what its own trace records say
    (last record's seg + 1; its terminal) and add up to the counters."""
    spec, _ = workloads.config(cfg)
    om = oracle_mod.OracleModel.from_spec(spec)
    n = 400
    r = om.run(n, seed=5, pid_begin=77, per_history=True, trace_cap=400 * n, max_segments=60)
    tr = r["trace"]
    idx = (tr["pid"] - 77).astype(np.int64)
    last = np.zeros(n, dtype=np.int64)
    term = np.zeros(n, dtype=np.int64)
    last[idx] = tr["seg"]
    term[idx] = tr["terminal"]
    capped = term == 4
    # a capped history's extra CAPPED record carries seg == nseg; every other last record is seg nseg-1
    assert np.array_equal(r["pnseg"].astype(np.int64), np.where(capped, last, last + 1))
    assert np.array_equal(r["pterm"].astype(np.int64), term)
    c = r["counters"]
    assert int(r["pnseg"].sum()) == c["segments"]
    assert [int((r["pterm"] == t).sum()) for t in (1, 2, 3, 4)] == \
        [c["absorptions"], c["leaks"], c["lost"], c["capped"]]
    assert c["capped"] > 0 and np.all(r["pterm"] > 0)
