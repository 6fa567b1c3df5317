"""Oracle pins for non-uniform rect arrays (Alg. 5 binary-search lattices, PAPER.md P:500-525 and
the footnote P:500-505; reading N1 in DESIGN.md): tile location against numpy's searchsorted on
the mesh divisions, wall-to-wall segment lengths, volume recovery (P9) on unequal tiles, and the
gap-column assembly reproducing the uniform C2 walk."""
import math

import numpy as np

import workloads
from workloads.models import Spec


def _slabs(oracle_mod, **kw):
    spec = workloads.models.nonuniform_slabs(**kw)
    lat = next(i for i, u in enumerate(spec["universes"]) if u["kind"] == "rect")
    return spec, oracle_mod.OracleModel.from_spec(spec), lat


def test_n1_index_matches_searchsorted(oracle_mod):
    """Tile i of axis a is the unique i with e[i] <= x < e[i+1]; -1 below e[0], n at or above
    e[n] (outer).  numpy.searchsorted(e, x, side='right') - 1 is the same definition."""
    spec, m, lat = _slabs(oracle_mod)
    edges = spec["universes"][lat]["edges"]
    rng = np.random.default_rng(11)
    pts = [rng.uniform([-1, -1, -1], [7, 4, 3]) for _ in range(3000)]
    pts += [np.array([x, y, z]) for x in edges[0] for y in edges[1] for z in edges[2]]   # exact edges
    for r in pts:
        ok, ijk, d, t, fl = m.locate_array(lat, tuple(r))
        want = [int(np.searchsorted(edges[a], r[a], side="right")) - 1 for a in range(3)]
        assert list(ijk) == want
        inside = all(0 <= want[a] < len(edges[a]) - 1 for a in range(3))
        assert ok == inside                          # no outer universe: outside tiles are LOST
        if inside:
            # the daughter frame: the point lies within half a tile width of the translation
            for a in range(3):
                w = edges[a][want[a] + 1] - edges[a][want[a]]
                assert -w / 2 - 1e-12 <= r[a] - t[a] < w / 2 + 1e-12
        on_edge = any(abs(r[a] - e) <= 1e-10 for a in range(3) for e in edges[a])
        assert bool(fl & 1) == on_edge               # F1 proximity to a mesh division


def test_n1_wall_to_wall_segments(oracle_mod):
    """A +x ray in a void non-uniform lattice: segments are the tile widths (1, 2, 3), then the
    reflective wall sends it back through the same tiles."""
    spec, m, lat = _slabs(oracle_mod, sigma_t=0.0, sigma_a=0.0)
    st = np.array([[0.5], [0.25], [0.35], [1.0], [0.0], [0.0]])
    res = m.run(1, states=st, trace_cap=64, max_segments=6)
    tr = res["trace"]
    assert np.array_equal(tr["s"][:6], [0.5, 2.0, 3.0, 3.0, 2.0, 1.0])
    assert list(tr["kind"][:6]) == [0, 0, 1, 0, 0, 1]       # cross, cross, reflect, cross, cross, reflect
    assert list(tr["level"][:6]) == [1, 1, 0, 1, 1, 0]


def test_n1_volume_recovery(oracle_mod):
    """P9 on unequal tiles: E[L_tile] / E[L_total] = V_tile / V_box (uniform medium, reflective)."""
    spec, m, lat = _slabs(oracle_mod)
    ex, ey, ez = spec["universes"][lat]["edges"]
    vol = np.array([(ex[i + 1] - ex[i]) * (ey[j + 1] - ey[j]) * (ez[k + 1] - ez[k])
                    for k in range(2) for j in range(2) for i in range(3)])
    exact = vol / vol.sum()
    B, nb = 20, 400
    fr = []
    for b in range(B):
        res = m.run(nb, seed=3, pid_begin=b * nb)
        fr.append(res["len"] / res["len"].sum())
    fr = np.array(fr)
    mean, se = fr.mean(0), fr.std(0, ddof=1) / math.sqrt(B)
    assert (np.abs(mean - exact) < 4.5 * se + 1e-4).all(), (mean, exact, se)


def test_n1_gap_lattice_bit_identical_to_uniform(oracle_mod):
    """A uniform lattice whose `outer` fills the water gap, and the same geometry as a
    non-uniform lattice with explicit gap columns: with dyadic divisions the tile centres are
    exact in both forms, so the walks are bit-identical (the gap walls coincide with the
    reflective box, where the root level wins the tie, O13)."""
    a = oracle_mod.OracleModel.from_spec(workloads.models.gap_lattice(False))
    b = oracle_mod.OracleModel.from_spec(workloads.models.gap_lattice(True))
    ra = a.run(500, seed=5, trace_cap=200000, pflags=True)
    rb = b.run(500, seed=5, trace_cap=200000, pflags=True)
    assert ra["counters"] == rb["counters"] and ra["counters"]["crossings"] > 10000
    for f in ("pid", "seg", "kind", "level", "j", "cell_before", "cell_after", "terminal", "flags", "s"):
        assert np.array_equal(ra["trace"][f], rb["trace"][f]), f
    assert np.array_equal(ra["out"], rb["out"])


def test_n1_gap_assembly_same_events_as_c2(oracle_mod):
    """C2 with explicit 0.04 cm gap columns (19x19 non-uniform): C2's walls and materials, so the
    event sequence is C2's.  The tile centres round differently ((e_i + e_i+1)/2 vs
    ll + (i + 1/2) p), which perturbs pin-frame coordinates by ulps; lengths agree closely."""
    a = oracle_mod.OracleModel.from_spec(workloads.config("c2")[0])
    b = oracle_mod.OracleModel.from_spec(workloads.models.c2_gap_assembly())
    ra = a.run(300, seed=5, trace_cap=100000, pflags=True)
    rb = b.run(300, seed=5, trace_cap=100000, pflags=True)
    assert ra["counters"] == rb["counters"]
    for f in ("pid", "seg", "kind", "level", "j", "cell_before", "cell_after", "terminal", "flags"):
        assert np.array_equal(ra["trace"][f], rb["trace"][f]), f
    assert np.allclose(ra["len"], rb["len"], rtol=1e-6, atol=0)


def test_n1_rejects_bad_edges(oracle_mod):
    sp = Spec("bad")
    root = sp.csg("root")
    box = workloads.models._box(sp, (0, 0, 0), (1, 1, 1), "vacuum")
    mt = sp.mat("m", 1.0, 0.5)
    t = sp.csg("t")
    sp.cell(t, [], material=mt)
    lat = sp.rect_edges("lat", [[0.0, 0.5, 0.5, 1.0], [0.0, 1.0], []], [t, t, t], None)   # repeated edge
    sp.cell(root, box, fill=lat)
    sp.root = root
    sp.source = {"lo": [0, 0, 0], "hi": [1, 1, 1]}
    try:
        oracle_mod.OracleModel.from_spec(sp.to_dict())
    except ValueError:
        return
    raise AssertionError("non-increasing edges accepted")
