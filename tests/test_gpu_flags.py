"""GPU parity of the O16 flags and the §8(c)4 flagged-history exclusion, on models built to fire
them (workloads.near_coincident / grazing_lattice; PAPER.md:554-556 coincident surfaces):

* F1 proximity of point location (nt_find_cells) equals the oracle's and the closed form, for
  every surface kind and both array kinds;
* traces and per-history flags of random batches equal the oracle's bit for bit, with flagged > 0
  on both sides, under every scheduler;
* F2 from the collision distance near a wall (explicit births, nt_track_states);
* per-cell totals after removing the union of flagged pids (re-run alone on both sides and
  subtracted: tests/parity_harness.py) agree within 1e-9, counters and exits exactly.
"""
import numpy as np
import pytest

import workloads
from parity_harness import compare_excluding_flagged, gpu_side, oracle_side
from test_oracle_flags import DC_DELTAS, F1, F2, _near_points, dc_wall_states

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

SCHEDS = ["block", "rounds", "warp", "history", "dp"]
FLAG_MODELS = {
    "near_cz": lambda: workloads.near_coincident("CZ"),
    "near_sphere": lambda: workloads.near_coincident("SPHERE"),
    "near_plane": lambda: workloads.near_coincident("PLANE"),
    "grazing_lattice": lambda: workloads.grazing_lattice(),
}


@pytest.fixture(scope="module")
def nt():
    import __graft_entry__
    __graft_entry__.build()
    import paper_2406_13849_b200 as nt
    assert torch.cuda.is_available()
    return nt


def test_find_cells_flags_parity(nt, oracle_mod):
    """nt_find_cells' F1 bits equal the oracle's and the closed form (5e-11 flags, 5e-10 does not)."""
    import math
    cases = []
    for kind in ("CZ", "SPHERE", "PLANE"):
        spec = workloads.near_coincident(kind, gap=1e-6)
        for delta, want in ((5e-11, F1), (-5e-11, F1), (1.3e-10, 0), (5e-10, 0)):
            cases.append((spec, _near_points(kind, delta), want))
    spec = workloads.grazing_lattice(gap=1e-3)
    for delta, want in ((5e-11, F1), (-5e-11, F1), (5e-10, 0)):
        cases.append((spec, [(0.625 + delta, 0.9, 5.0), (-0.9, -0.625 + delta, 3.0)], want))
    for orient, base in (("pointy", 0.0), ("flat", 30.0)):
        spec = workloads.hex_pins_small(orient)
        for delta, want in ((5e-11, F1), (1.3e-10, 0)):
            pts = []
            for k in range(6):
                a = math.radians(base + 60.0 * k)
                n = np.array([math.cos(a), math.sin(a)])
                xy = np.array([0.1, -0.05]) + (0.8 + delta) * n + 0.13 * np.array([-n[1], n[0]])
                pts.append((xy[0], xy[1], 1.7))
            cases.append((spec, pts, want))
    models = {}
    for spec, pts, want in cases:
        if spec["name"] not in models:
            models[spec["name"]] = (nt.Model.from_spec(spec, device=0), oracle_mod.OracleModel.from_spec(spec))
        m, om = models[spec["name"]]
        xyz = np.array(pts, dtype=np.float64).T.copy()
        cell, fl = m.find_cells(torch.tensor(xyz, device="cuda"))
        torch.cuda.synchronize()
        oc, of = om.find_cells(xyz)
        assert np.array_equal(cell.cpu().numpy(), oc)
        assert np.array_equal(fl.cpu().numpy(), of)
        assert np.all(of == want), (spec["name"], pts, of, want)


@pytest.mark.parametrize("sched", SCHEDS)
@pytest.mark.parametrize("name", list(FLAG_MODELS))
def test_flag_models_trace_parity(nt, oracle_mod, name, sched):
    """Random births in the near-coincident models: traces (with their sticky flags), per-history
    flags, counters and tallies bit-exact vs the oracle; both sides flag > 0 histories."""
    spec = FLAG_MODELS[name]()
    m = nt.Model.from_spec(spec, device=0)
    om = oracle_mod.OracleModel.from_spec(spec)
    n, seed = 3000, 4
    cap = 300 * n
    res = m.track(n, seed=seed, pflags=True, trace_cap=cap, scheduler=sched)
    torch.cuda.synchronize()
    g = m.unpack(res["out"])
    o = om.run(n, seed=seed, pflags=True, trace_cap=cap)
    gpf = res["pflags"].cpu().numpy()[:n]
    assert np.array_equal(gpf, o["pflags"])
    assert g["counters"] == o["counters"]
    assert g["counters"]["flagged"] > 0 and int((gpf != 0).sum()) == g["counters"]["flagged"]
    assert np.array_equal(g["exits"], o["exits"])
    assert np.allclose(g["len"], o["len"], rtol=1e-12, atol=0)
    gt, ot = nt.Model.trace_records(res), o["trace"]
    assert len(gt) == len(ot)
    for f in ("pid", "seg", "kind", "level", "j", "cell_before", "cell_after", "terminal", "flags", "s"):
        assert np.array_equal(gt[f], ot[f]), f
    # both kinds of flag fire in every model
    assert np.any(gpf & F1) and np.any(gpf & F2)


@pytest.mark.parametrize("sched", SCHEDS)
def test_dc_near_wall_flags(nt, oracle_mod, sched):
    """F2 from |d_c - d_s| <= 1e-10 (explicit births a tuned distance before a wall): GPU flags equal
    the oracle's and the closed form; the first event is the collision iff the wall is beyond d_c."""
    spec = workloads.infinite_medium(1.0, 0.25)
    st, dl = dc_wall_states(oracle_mod, 11, 280, DC_DELTAS)
    n = st.shape[1]
    m = nt.Model.from_spec(spec, device=0)
    res = m.track(n, seed=11, pflags=True, states=torch.tensor(st, device="cuda"), scheduler=sched)
    torch.cuda.synchronize()
    gpf = res["pflags"].cpu().numpy()[:n]
    o = oracle_mod.OracleModel.from_spec(spec).run(n, seed=11, states=st, pflags=True)
    assert np.array_equal(gpf, o["pflags"])
    for i, d in enumerate(dl):
        if d is not None:
            assert gpf[i] == (F2 if abs(d) <= 1e-10 else 0)


@pytest.mark.parametrize("name", list(FLAG_MODELS))
def test_flagged_exclusion_harness(nt, oracle_mod, name):
    """§8(c)4: union of flagged pids, re-run alone on both sides, subtracted; the rest agrees
    (counters and exits exact, len within 1e-9).  5-90 % of these histories are flagged, so the
    union is re-run in thousands of contiguous pid runs."""
    spec = FLAG_MODELS[name]()
    m = nt.Model.from_spec(spec, device=0)
    om = oracle_mod.OracleModel.from_spec(spec)
    rep = compare_excluding_flagged(gpu_side(m, 9), oracle_side(om, 9), m.n_mc, 20_000, pid_begin=1000)
    assert rep["flagged_gpu"] > 0 and rep["flags_equal"]
    assert rep["union"] == rep["flagged_gpu"]


def test_flagged_exclusion_harness_states(nt, oracle_mod):
    """The harness with explicit births (nt_track_states): flagged d_c-near-wall histories removed."""
    spec = workloads.infinite_medium(1.0, 0.25)
    st, _ = dc_wall_states(oracle_mod, 11, 280, DC_DELTAS)
    m = nt.Model.from_spec(spec, device=0)
    om = oracle_mod.OracleModel.from_spec(spec)
    rep = compare_excluding_flagged(gpu_side(m, 11, states=st), oracle_side(om, 11, states=st), m.n_mc,
                                    st.shape[1])
    assert rep["flagged_gpu"] > 0 and rep["flags_equal"]
