"""Oracle geometry pins: P3 analytic distances, P4 sense/containment, P5 rect index,
P6 hex index (worked values + Voronoi brute force), P7 brute-force location, P16 partition."""
import math
import os

import numpy as np
import pytest

import workloads
from workloads.models import Spec

INF = float("inf")
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _surface_model(oracle_mod):
    sp = Spec("surfaces")
    ids = {
        "px1": sp.surf("PX", [1.0]),
        "cz1": sp.surf("CZ", [0.0, 0.0, 1.0]),
        "cz5": sp.surf("CZ", [0.0, 0.0, 5.0]),
        "sph2": sp.surf("SPHERE", [0.0, 0.0, 0.0, 2.0]),
        "pl": sp.surf("PLANE", [1.0, 1.0, 0.0, 1.0]),
        "pz0": sp.surf("PZ", [0.0]),
        "czoff": sp.surf("CZ", [0.3, -0.7, 1.7]),
        "sphoff": sp.surf("SPHERE", [0.2, 0.1, -0.4, 1.1]),
        "pltilt": sp.surf("PLANE", [0.3, -0.4, 0.5, 0.25]),
    }
    root = sp.csg("root")
    m = sp.mat("m", 1.0, 0.5)
    sp.cell(root, [], material=m)
    sp.root = root
    sp.source = {"lo": [0, 0, 0], "hi": [1, 1, 1]}
    return oracle_mod.OracleModel.from_spec(sp.to_dict()), ids


def test_p3_analytic_distances(oracle_mod):
    """P3: closed-form distances, cell-aware O11."""
    m, I = _surface_model(oracle_mod)
    d = m.surface_distance
    X, Y, Z = (1, 0, 0), (0, 1, 0), (0, 0, 1)
    assert d(I["px1"], False, (0, 0, 0), X) == 1.0
    assert d(I["px1"], False, (0, 0, 0), Y) == INF
    assert d(I["px1"], False, (0, 0, 0), (-1, 0, 0)) == INF
    assert d(I["cz1"], False, (0, 0, 0), X) == 1.0
    assert d(I["cz1"], True, (-2, 0, 0), X) == 1.0
    assert d(I["cz1"], False, (1, 0, 0), (-1, 0, 0), onsurf=True) == 2.0
    assert d(I["cz1"], False, (0, 0, 0), Z) == INF
    assert d(I["cz1"], True, (-2, 1, 0), X) == 2.0          # tangent is a hit
    assert d(I["cz5"], False, (0, 0, 0), (0.6, 0.8, 0)) == 5.0
    assert d(I["cz5"], False, (3, 0, 0), Y) == 4.0
    assert d(I["sph2"], False, (0, 0, 0), Z) == 2.0
    assert d(I["sph2"], True, (0, 0, -5), Z) == 3.0
    assert d(I["pl"], False, (0, 0, 0), X) == 1.0
    # outside moving away / missing: no exit
    assert d(I["cz1"], True, (2, 0, 0), X) == INF
    assert d(I["cz1"], True, (-2, 1.5, 0), X) == INF


def test_p3_random_rays_hit_the_surface(oracle_mod):
    """For random rays, the returned d puts the point on the surface (|f| ~ 0) and the sense
    changes across it; an infinite d means the sense never changes along the ray."""
    m, I = _surface_model(oracle_mod)
    rng = np.random.default_rng(3)
    for name in ("czoff", "sphoff", "pltilt", "cz5", "sph2"):
        sid = I[name]
        for _ in range(120):
            r = rng.uniform(-3, 3, 3)
            om = rng.normal(size=3)
            om /= np.linalg.norm(om)
            f0 = m.surface_f(sid, r)
            sense_pos = f0 >= 0.0
            dist = m.surface_distance(sid, sense_pos, r, om)
            ts = np.linspace(1e-6, 12.0, 1200)
            fs = np.array([m.surface_f(sid, r + t * om) for t in ts])
            flips = np.nonzero((fs >= 0.0) != sense_pos)[0]
            if dist == INF:
                assert len(flips) == 0
            else:
                scale = 1.0 + np.abs(r).max() ** 2
                assert abs(m.surface_f(sid, r + dist * om)) < 1e-12 * scale
                if len(flips):
                    assert dist <= ts[flips[0]] + 1e-9
                    assert dist >= ts[max(flips[0] - 1, 0)] - 1e-9


def test_p4_sense(oracle_mod):
    """P4: sign of the implicit function, f = 0 -> positive (O4)."""
    m, I = _surface_model(oracle_mod)
    assert m.surface_f(I["px1"], (2, 0, 0)) > 0
    assert m.surface_f(I["cz1"], (0, 0, 5)) < 0
    assert m.surface_f(I["pz0"], (0, 0, 0)) == 0.0          # O4: f >= 0 is POS


def test_p4_containment(oracle_mod):
    """unit cube cell and a pin cell."""
    sp = Spec("cube")
    root = sp.csg("root")
    box = workloads.models._box(sp, (0, 0, 0), (1, 1, 1), "vacuum")
    cz = sp.surf("CZ", [0.5, 0.5, 0.3])
    m1 = sp.mat("a", 1, 0)
    sp.cell(root, box + [-(cz + 1)], material=m1)
    sp.cell(root, box + [cz + 1], material=m1)
    sp.root = root
    sp.source = {"lo": [0, 0, 0], "hi": [1, 1, 1]}
    m = oracle_mod.OracleModel.from_spec(sp.to_dict())
    cells, _ = m.find_cells(np.array([[0.5, 2.0, 0.9], [0.5, 0.5, 0.5], [0.5, 0.5, 0.5]]))
    assert list(cells) == [0, -1, 1]


def _rect_model(oracle_mod):
    sp = Spec("rect1d")
    root = sp.csg("root")
    box = workloads.models._box(sp, (-5, -0.5, -0.5), (5, 0.5, 0.5), "vacuum")
    m = sp.mat("m", 0, 0)
    inner = sp.csg("inner")
    sp.cell(inner, [], material=m)
    outer = sp.csg("outer")
    sp.cell(outer, [], material=m)
    lat = sp.rect("lat", (0.0, -0.5, 0.0), (1.0, 1.0, 0.0), (4, 1, 1), [inner] * 4, outer)
    sp.cell(root, box, fill=lat)
    sp.root = root
    sp.source = {"lo": [0, 0, 0], "hi": [1, 1, 1]}
    return oracle_mod.OracleModel.from_spec(sp.to_dict()), lat, inner, outer


def test_p5_rect_index(oracle_mod):
    """P5: LL=0, p=1: x=2.5 -> 2; x=1.0 -> 1 (tie to higher, O8);
    x=-0.5 -> -1 (outer, infinite tiling); tile centre LL+(i+0.5)p."""
    m, lat, inner, outer = _rect_model(oracle_mod)
    ok, ijk, d, t, fl = m.locate_array(lat, (2.5, 0.0, 0.0))
    assert ok and ijk[0] == 2 and d == inner and t[0] == 2.5
    ok, ijk, d, t, fl = m.locate_array(lat, (1.0, 0.0, 0.0))
    assert ijk[0] == 1 and fl == 1                       # on an edge: F1 proximity flag
    ok, ijk, d, t, fl = m.locate_array(lat, (-0.5, 0.0, 0.0))
    assert ijk[0] == -1 and d == outer and t[0] == -0.5
    ok, ijk, d, t, fl = m.locate_array(lat, (4.0, 0.0, 0.0))
    assert ijk[0] == 4 and d == outer
    rng = np.random.default_rng(4)
    for x in rng.uniform(-3, 7, 500):
        ok, ijk, d, t, fl = m.locate_array(lat, (x, 0.0, 0.0))
        assert ijk[0] == math.floor(x)                    # exact for LL=0, p=1


def test_p5_rect_crossing_walk(oracle_mod):
    """Alg. 6: a +x ray crosses every unit tile wall once; each segment is 1."""
    m, lat, inner, outer = _rect_model(oracle_mod)
    st = np.array([[-4.5], [0.0], [0.0], [1.0], [0.0], [0.0]])
    res = m.run(1, states=st, trace_cap=64)
    tr = res["trace"]
    # root-box wall at -5 is behind; tiles -5..4 walls at integers -4..4, then the box at +5
    lens = tr["s"]
    assert np.allclose(lens, [0.5] + [1.0] * 8 + [1.0], rtol=0, atol=1e-15)
    assert tr["kind"][-1] == 2                            # LEAK through the vacuum box


def _hex_model(oracle_mod, orient, pitch=2.0, center=(0.0, 0.0)):
    sp = Spec("hex")
    root = sp.csg("root")
    box = workloads.models._box(sp, (-20, -20, -1), (20, 20, 1), "vacuum")
    m = sp.mat("m", 1, 0)
    pins = []
    for k in range(19):
        u = sp.csg(f"p{k}")
        sp.cell(u, [], material=m)
        pins.append(u)
    outer = sp.csg("outer")
    sp.cell(outer, [], material=m)
    lat = sp.hex("lat", orient, center, pitch, 3, pins, outer)
    sp.cell(root, box, fill=lat)
    sp.root = root
    sp.source = {"lo": [0, 0, 0], "hi": [1, 1, 1]}
    return oracle_mod.OracleModel.from_spec(sp.to_dict()), lat, pins, outer


def _hex_centre(orient, p, q, r, C=(0.0, 0.0)):
    H = math.sqrt(3.0) / 2.0
    if orient == "pointy":
        a1, a2 = (p, 0.0), (p / 2, p * H)
    else:
        a1, a2 = (p * H, p / 2), (0.0, p)
    return (C[0] + q * a1[0] + r * a2[0], C[1] + q * a1[1] + r * a2[1])


def test_p6_hex_worked_values(oracle_mod):
    """P6: worked values (tests/golden/hex_worked_values.txt, reading O9)."""
    m, lat, pins, outer = _hex_model(oracle_mod, "pointy")
    with open(os.path.join(GOLDEN, "hex_worked_values.txt")) as f:
        rows = [ln.split() for ln in f if ln.strip() and not ln.startswith("#")]
    for x, y, q, r in rows:
        ok, ijk, d, t, fl = m.locate_array(lat, (float(x), float(y), 0.0))
        assert (ijk[0], ijk[1]) == (int(q), int(r)), (x, y, ijk)


@pytest.mark.parametrize("orient", ["pointy", "flat"])
def test_p6_hex_voronoi(oracle_mod, orient):
    """P6: away from boundaries the owning tile is the nearest tile centre (a hexagonal
    tiling is the Voronoi diagram of its centres) -- brute force over all centres."""
    p, C = 1.7, (0.3, -0.2)
    m, lat, pins, outer = _hex_model(oracle_mod, orient, p, C)
    tiles = workloads.hex_tiles(10)
    cents = np.array([_hex_centre(orient, p, q, r, C) for q, r in tiles])
    rng = np.random.default_rng(5)
    nchk = 0
    for x, y in rng.uniform(-7, 7, size=(3000, 2)):
        dd = np.hypot(cents[:, 0] - x, cents[:, 1] - y)
        o = np.argsort(dd)
        if dd[o[1]] - dd[o[0]] < 1e-9:
            continue
        ok, ijk, d, t, fl = m.locate_array(lat, (x, y, 0.0))
        assert (ijk[0], ijk[1]) == tiles[o[0]]
        nchk += 1
    assert nchk > 2900
    # every tile centre maps to itself; in-lattice tiles fill in O9 order, others -> outer
    ring3 = workloads.hex_tiles(3)
    for (q, r) in tiles:
        cx, cy = _hex_centre(orient, p, q, r, C)
        ok, ijk, d, t, fl = m.locate_array(lat, (cx, cy, 0.0))
        assert (ijk[0], ijk[1]) == (q, r)
        assert d == (pins[ring3.index((q, r))] if (q, r) in ring3 else outer)
        assert abs(t[0] - cx) < 1e-12 and abs(t[1] - cy) < 1e-12


@pytest.mark.parametrize("orient", ["pointy", "flat"])
def test_p6_hex_neighbours(oracle_mod, orient):
    """Points at 0.49p / 0.51p along each face normal map to self / neighbour delta_k."""
    p = 2.0
    m, lat, pins, outer = _hex_model(oracle_mod, orient, p)
    deltas = [(1, 0), (0, 1), (-1, 1), (-1, 0), (0, -1), (1, -1)]
    for (q0, r0) in workloads.hex_tiles(3):
        cx, cy = _hex_centre(orient, p, q0, r0)
        for k, (dq, dr) in enumerate(deltas):
            nx, ny = _hex_centre(orient, p, q0 + dq, r0 + dr)
            ux, uy = (nx - cx) / p, (ny - cy) / p
            ok, ijk, *_ = m.locate_array(lat, (cx + 0.49 * p * ux, cy + 0.49 * p * uy, 0.0))
            assert (ijk[0], ijk[1]) == (q0, r0)
            ok, ijk, *_ = m.locate_array(lat, (cx + 0.51 * p * ux, cy + 0.51 * p * uy, 0.0))
            assert (ijk[0], ijk[1]) == (q0 + dq, r0 + dr)


def test_p7_pincell_location(oracle_mod):
    """P7: pincell cell by rho^2 vs r_i^2 (closed form) equals the oracle's descent."""
    spec = workloads.c1_pincell()
    m = oracle_mod.OracleModel.from_spec(spec)
    rng = np.random.default_rng(6)
    pts = np.stack([rng.uniform(-0.63, 0.63, 5000), rng.uniform(-0.63, 0.63, 5000),
                    rng.uniform(0, 365.76, 5000)])
    cells, fl = m.find_cells(pts)
    rho2 = pts[0] ** 2 + pts[1] ** 2
    radii = workloads.models.PIN_R
    cls = np.searchsorted(np.array(radii) ** 2, rho2, side="right")
    # pin cells are global cells 1..4 (cell 0 is the root box cell)
    assert np.array_equal(cells, cls + 1)
    assert not fl.any()


def test_p7_lattice_location(oracle_mod):
    """P7: 3x3 lattice -- tile by floor and annulus by rho^2 reproduce the material."""
    spec = workloads.lattice3_nested()
    m = oracle_mod.OracleModel.from_spec(spec)
    rng = np.random.default_rng(7)
    p, ll = 1.25, -1.875
    pts = np.stack([rng.uniform(ll, -ll, 5000), rng.uniform(ll, -ll, 5000), rng.uniform(0, 10, 5000)])
    cells, fl = m.find_cells(pts)
    i = np.floor((pts[0] - ll) / p)
    j = np.floor((pts[1] - ll) / p)
    cx, cy = ll + (i + 0.5) * p, ll + (j + 0.5) * p
    rho2 = (pts[0] - cx) ** 2 + (pts[1] - cy) ** 2
    cls = np.searchsorted(np.array(workloads.models.PIN_R) ** 2, rho2, side="right")
    mats = np.array([m.cell_material(c) for c in cells])
    assert np.array_equal(mats, np.array([0, 1, 2, 3])[cls])


@pytest.mark.parametrize("cfg", ["c1", "c2", "c3", "c4", "c5m", "c5r"])
def test_p16_partition(oracle_mod, cfg):
    """P16: random points are contained by exactly one cell of each CSG
    universe (root universe over the source box; pin universes over their tile)."""
    spec, _ = workloads.config(cfg)
    m = oracle_mod.OracleModel.from_spec(spec)
    rng = np.random.default_rng(8)
    lo, hi = np.array(spec["source"]["lo"]), np.array(spec["source"]["hi"])
    root = spec["root"]
    for r in rng.uniform(lo, hi, size=(300, 3)):
        assert m.count_containing(root, r) <= 1
    for uid, u in enumerate(spec["universes"]):
        if u["kind"] != "csg" or uid == root:
            continue
        for r in rng.uniform(-0.6, 0.6, size=(200, 3)):
            assert m.count_containing(uid, r) == 1
    # every source point is located (no gaps inside the model)
    pts = rng.uniform(lo, hi, size=(2000, 3)).T.copy()
    cells, fl = m.find_cells(pts)
    assert (cells >= 0).all()


@pytest.mark.parametrize("orient", ["pointy", "flat"])
@pytest.mark.parametrize("pitch", [2.0, 1.26, 9.0, 30.0])
def test_o9_hex_faces_exact_partition(oracle_mod, orient, pitch):
    """O9 s-space membership is an exact partition on faces: adjacent tiles compare s_k with the
    same rounded bound p (m_k + 1/2), so a point on (or an ulp off) a shared face belongs to exactly
    one tile of the window.  Points up to 0.28 p from the face's mid-point (the half side is p / (2 sqrt 3)
    = 0.2887 p, so vertices are excluded)."""
    C = (0.37, -0.21)
    m, lat, pins, outer = _hex_model(oracle_mod, orient, pitch, C)
    deltas = [(1, 0), (0, 1), (-1, 1), (-1, 0), (0, -1), (1, -1)]
    rng = np.random.default_rng(11)
    n = 0
    for (q0, r0) in workloads.hex_tiles(3):
        cx, cy = _hex_centre(orient, pitch, q0, r0, C)
        for (dq, dr) in deltas:
            nx, ny = _hex_centre(orient, pitch, q0 + dq, r0 + dr, C)
            ux, uy = (nx - cx) / pitch, (ny - cy) / pitch
            for a in rng.uniform(-0.28, 0.28, size=6) * pitch:
                x = cx + 0.5 * pitch * ux - a * uy
                y = cy + 0.5 * pitch * uy + a * ux
                for xx in (x, np.nextafter(x, np.inf), np.nextafter(x, -np.inf)):
                    owners = [(q, r) for q in range(q0 - 3, q0 + 4) for r in range(r0 - 3, r0 + 4)
                              if m.hex_owns(lat, q, r, (xx, y, 0.0))]
                    assert len(owners) == 1, (orient, pitch, (q0, r0), (dq, dr), owners)
                    assert owners[0] in ((q0, r0), (q0 + dq, r0 + dr))
                    n += 1
    assert n > 1000
