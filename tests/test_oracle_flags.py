"""Oracle pins of the O16 flags (the north star's "rays flagged within 1e-10 cm
of a coincident surface"; PAPER.md:554-556 on coincident surfaces), against closed forms:

* F1 proximity at a descended level, for every surface kind and array kind: a point at distance
  5e-11 cm from a surface / rect wall / hex face is flagged, one at 5e-10 cm is not;
* F1 on the far side of a crossing, and F2 near-ties between two surfaces of one cell, between a CSG
  surface and a lattice wall one level up, and between a wall and the collision distance d_c;
  each on deterministic rays whose distances are known in closed form, with controls just outside
  the 1e-10 cm band.
"""
import math

import numpy as np
import pytest

import workloads

F1, F2, F3 = 1, 2, 4
CROSS, REFLECT, LEAK, COLLIDE = 0, 1, 2, 3


def _unit(v):
    v = np.asarray(v, dtype=np.float64)
    return v / np.linalg.norm(v)


def _near_points(kind, delta):
    """Points at signed distance `delta` outside the body surface S of workloads.near_coincident."""
    R = workloads.NEAR_BODY
    if kind == "CZ":
        return [(R + delta, 0.0, 0.1), (0.0, -(R + delta), -0.3),
                ((R + delta) * 0.6, (R + delta) * 0.8, 0.7)]
    if kind == "SPHERE":
        return [tuple((R + delta) * _unit(d)) for d in ((1, 0, 0), (1, 1, 1), (-0.3, 0.5, -0.8))]
    n = _unit(workloads.NEAR_PLANE_N)
    t1 = _unit(np.cross(n, (0.0, 0.0, 1.0)))
    return [tuple((R + delta) * n + a * t1) for a in (0.0, 0.2, -0.35)]


@pytest.mark.parametrize("kind", ["CZ", "SPHERE", "PLANE"])
def test_f1_proximity_quadrics_and_planes(oracle_mod, kind):
    """F1 at a CSG level: |f| <= 1e-10 x |grad f| scale (CZ / SPHERE: 2R; PLANE: |n|), i.e. the
    point is within 1e-10 cm of the surface.  S' is 1e-6 cm away here, so only S can fire.  R = 0.3
    and |n| = 3, so an unscaled |f| <= 1e-10 would flag at 1.3e-10 cm (CZ / SPHERE) and miss 5e-11
    (PLANE)."""
    om = oracle_mod.OracleModel.from_spec(workloads.near_coincident(kind, gap=1e-6))
    for delta, want in ((5e-11, F1), (-5e-11, F1), (0.9e-10, F1), (-0.9e-10, F1),
                        (1.3e-10, 0), (-1.3e-10, 0), (5e-10, 0), (-5e-10, 0), (2e-10, 0)):
        pts = np.array(_near_points(kind, delta)).T
        cells, fl = om.find_cells(pts)
        assert np.all(fl == want), (kind, delta, fl)
        assert np.all(cells == (1 if delta > 0 else 0))


def test_f1_proximity_axis_plane(oracle_mod):
    """F1 for an axis plane (tolerance 1e-10): the vacuum box wall x = 1."""
    om = oracle_mod.OracleModel.from_spec(workloads.near_coincident("CZ", gap=1e-6))
    for delta, want in ((5e-11, F1), (0.9e-10, F1), (5e-10, 0), (1e-9, 0)):
        pts = np.array([(1.0 - delta, 0.9, 0.2), (-1.0 + delta, 0.8, -0.6), (0.9, 0.9, 1.0 - delta)]).T
        _, fl = om.find_cells(pts)
        assert np.all(fl == want), (delta, fl)


def test_f1_proximity_rect_wall(oracle_mod):
    """F1 at a rect level: |x - e(i)| <= 1e-10 for the lattice edge e = -1.875 + 2 x 1.25 = 0.625."""
    om = oracle_mod.OracleModel.from_spec(workloads.grazing_lattice(gap=1e-3))
    for delta, want in ((5e-11, F1), (-5e-11, F1), (5e-10, 0), (-5e-10, 0)):
        pts = np.array([(0.625 + delta, 0.9, 5.0), (-0.9, -0.625 + delta, 3.0)]).T
        _, fl = om.find_cells(pts)
        assert np.all(fl == want), (delta, fl)


@pytest.mark.parametrize("orient", ["pointy", "flat"])
def test_f1_proximity_hex_face(oracle_mod, orient):
    """F1 at a hex level: p |t_k - (m_k +- 1/2)| <= 1e-10, i.e. the point is within 1e-10 cm of a
    face of its tile (t-space of O9).  Faces of tile (0, 0) of hex_pins_small (C = (0.1, -0.05),
    pitch 1.6): apothem 0.8 along the face normals (POINTY: 0 deg, 60 deg, ...; FLAT: 30 deg, ...)."""
    om = oracle_mod.OracleModel.from_spec(workloads.hex_pins_small(orient))
    C = np.array([0.1, -0.05])
    base = 0.0 if orient == "pointy" else 30.0
    for delta, want in ((5e-11, F1), (-5e-11, F1), (1.3e-10, 0), (-1.3e-10, 0), (5e-10, 0), (-5e-10, 0)):
        pts = []
        for k in range(6):
            a = math.radians(base + 60.0 * k)
            nrm = np.array([math.cos(a), math.sin(a)])
            tang = np.array([-nrm[1], nrm[0]])
            xy = C + (0.8 + delta) * nrm + 0.13 * tang
            pts.append((xy[0], xy[1], 1.7))
        _, fl = om.find_cells(np.array(pts).T)
        assert np.all(fl == want), (orient, delta, fl)


def _trace_of(om, states, max_segments=64):
    n = states.shape[1]
    res = om.run(n, seed=3, states=states, pflags=True, trace_cap=200 * n, max_segments=max_segments)
    return res, res["trace"]


def _ray_states(rays):
    st = np.zeros((6, len(rays)))
    for i, (r, d) in enumerate(rays):
        st[:3, i] = r
        st[3:, i] = _unit(d)
    return st


def _normal_and_start(kind):
    """Outward normal at the surface point the test rays cross, and that point."""
    R = workloads.NEAR_BODY
    if kind == "CZ":
        n = np.array([1.0, 0.0, 0.0])
    elif kind == "SPHERE":
        n = _unit((1.0, 1.0, 1.0))
    else:
        n = _unit(workloads.NEAR_PLANE_N)
    return n, R * n


@pytest.mark.parametrize("kind", ["CZ", "SPHERE", "PLANE"])
def test_f1_f2_coincident_pair_rays(oracle_mod, kind):
    """Void model, deterministic rays (closed-form distances):
    out: from inside the body along the outward normal -> crossing S is flagged F1 (the new cell has S'
         5e-11 away), not F2 (S' is behind);
    in:  from outside along the inward normal -> the first segment has S at d and S' at d + 5e-11 ->
         F2 before any F1;
    oblique in: entering at cos(theta) = 0.4 puts S' 5e-11 / 0.4 = 1.25e-10 cm further along the
         ray (planes; ~1.15e-10 for the curved surfaces at impact parameter 0.9 R) -> no F2;
    control model (S' 5e-10 away): no flag on any ray."""
    n, p0 = _normal_and_start(kind)
    t = _unit(np.cross(n, (0.3, 0.1, 0.9)))
    rays = [(p0 - 0.3 * n, n),                          # out
            (p0 + 0.4 * n, -n)]                         # in
    if kind == "PLANE":
        d = -0.4 * n + math.sqrt(1 - 0.16) * t          # cos = 0.4 against the inward normal
        rays.append((p0 - 0.2 * d, d))
    else:
        # impact parameter b = 0.9 R: S' lies 5e-11 R / sqrt(R^2 - b^2) ~ 1.15e-10 cm beyond S
        b = 0.9 * workloads.NEAR_BODY
        tt = t if kind == "SPHERE" else np.array([0.0, 1.0, 0.0])
        # a line at distance b from the axis/centre, entering through S
        start = b * tt + 0.9 * np.array([1.0, 0.0, 0.0]) if kind == "CZ" else b * tt + 0.9 * n
        dirn = np.array([-1.0, 0.0, 0.0]) if kind == "CZ" else -n
        rays.append((start, dirn))
    om = oracle_mod.OracleModel.from_spec(workloads.near_coincident(kind, void=True))
    res, tr = _trace_of(om, _ray_states(rays))
    body = 0
    # out
    r0 = tr[tr["pid"] == 0]
    assert r0[0]["kind"] == CROSS and r0[0]["cell_before"] == body and r0[0]["cell_after"] == 1
    assert r0[0]["flags"] == F1
    assert abs(r0[0]["s"] - workloads.NEAR_BODY) <= 1e-15
    # in
    r1 = tr[tr["pid"] == 1]
    assert r1[0]["kind"] == CROSS and r1[0]["cell_after"] == body and r1[0]["flags"] == F2
    assert abs(r1[0]["s"] - 0.4) <= 1e-15
    # oblique in: no F2 on entry; F1 once it leaves the body through S (curved surfaces)
    r2 = tr[tr["pid"] == 2]
    entry = np.nonzero(r2["cell_after"] == body)[0][0]
    assert r2[entry]["flags"] & F2 == 0
    if kind != "PLANE":
        exit_ = np.nonzero((r2["cell_before"] == body) & (r2["kind"] == CROSS))[0][0]
        assert r2[exit_]["flags"] & F1
    assert np.all(res["pflags"][:2] == [F1, F1 | F2] if kind != "PLANE" else res["pflags"][:2] == [F1, F2])
    # control: S' 5e-10 cm inside S
    omc = oracle_mod.OracleModel.from_spec(workloads.near_coincident(kind, gap=5e-10, void=True))
    resc, _ = _trace_of(omc, _ray_states(rays))
    assert np.all(resc["pflags"] == 0)


def test_f2_across_levels_grazing_lattice(oracle_mod):
    """A CSG plane 5e-11 cm inside a lattice wall one level up (void lattice, deterministic +x ray
    from the middle tile): the first segment has the plane at 0.325 - 5e-11 and the wall at 0.325,
    so it is F2 (not F1); the ray's first descent into a tile through its +x wall, moving -x after
    the box reflection, lands 5e-11 from the plane: F1 from then on.  Control: 5e-10 -> no flags."""
    st = _ray_states([((0.3, 0.55, 5.0), (1.0, 0.0, 0.0))])
    om = oracle_mod.OracleModel.from_spec(workloads.grazing_lattice(void=True))
    res, tr = _trace_of(om, st, max_segments=12)
    assert tr[0]["kind"] == CROSS and tr[0]["level"] == 2 and tr[0]["flags"] == F2
    assert abs(tr[0]["s"] - (0.325 - 5e-11)) <= 1e-15
    # entering a tile through its +x wall (lattice level 1, moving -x: wall j = x- = 0)
    k = np.nonzero((tr["level"] == 1) & (tr["j"] == 0) & (tr["kind"] == CROSS))[0][0]
    assert np.all(tr[:k]["flags"] & F1 == 0)
    assert tr[k]["flags"] & F1
    omc = oracle_mod.OracleModel.from_spec(workloads.grazing_lattice(gap=5e-10, void=True))
    resc, trc = _trace_of(omc, st, max_segments=12)
    assert np.all(trc["flags"] & (F1 | F2) == 0)
    assert resc["pflags"][0] == F3                      # capped at 12 segments, nothing else


def dc_wall_states(oracle_mod, seed, n, deltas):
    """Explicit births in the infinite-medium box (Sigma_t = 1, REFLECT walls at +-1): particle i
    starts at x = 1 - (tau_i + delta), moving +x, where tau_i = -ln xi_tau (epoch 0, block 0, O17)
    is its first collision distance (d_c = tau / Sigma_t = tau).  The wall is then delta beyond
    d_c (delta > 0) or before it (delta < 0).  Returns (states, delta per particle, kept pids)."""
    key = [seed & 0xFFFFFFFF, seed >> 32]
    rows, dl = [], []
    pid = 0
    while len(rows) < n:
        x = oracle_mod.philox([pid, 0, 0, 0], key)
        tau = -oracle_mod.log(oracle_mod.u01(int(x[2]), int(x[3])))
        if tau < 1.5:
            d = deltas[len(rows) % len(deltas)]
            rows.append((1.0 - (tau + d), 0.1, -0.2, 1.0, 0.0, 0.0))
            dl.append(d)
        else:
            rows.append((0.0, 0.0, 0.0, 0.0, 0.0, 1.0))  # placeholder history, not tuned
            dl.append(None)
        pid += 1
    return np.array(rows).T.copy(), dl


DC_DELTAS = (5e-11, -5e-11, 0.9e-10, -0.9e-10, 3e-10, -3e-10, 1e-6)


def test_f2_collision_distance_near_wall(oracle_mod):
    """F2 with d_c: 0 < |d_c - d_s| <= 1e-10 flags (d_c = tau exactly, since Sigma_t = 1; d_s = 1 - x0
    to within an ulp of tau).  |delta| = 3e-10 and 1e-6 do not flag (the first event; later events
    flag only by chance, with probability ~1e-10 each)."""
    om = oracle_mod.OracleModel.from_spec(workloads.infinite_medium(1.0, 0.25))
    st, dl = dc_wall_states(oracle_mod, 11, 280, DC_DELTAS)
    res = om.run(st.shape[1], seed=11, states=st, pflags=True, trace_cap=20000)
    tr = res["trace"]
    n_tuned = 0
    for i, d in enumerate(dl):
        if d is None:
            continue
        n_tuned += 1
        want = F2 if abs(d) <= 1e-10 else 0
        assert res["pflags"][i] == want, (i, d, res["pflags"][i])
        first = tr[(tr["pid"] == i)][0]
        # the first event is the collision when the wall is beyond d_c, the reflection otherwise
        assert first["kind"] == (COLLIDE if d > 0 else REFLECT)
    assert n_tuned >= 50
