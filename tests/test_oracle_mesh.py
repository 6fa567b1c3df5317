"""Oracle pins for the superimposed Cartesian mesh track-length tally (PAPER.md
P:1006-1008 and P:1404-1407; reading M1 in DESIGN.md): single rays against a brute-force
numerical integration along the ray, conservation (the mesh tally of a mesh that covers the model
equals the cell tally), and voxel-volume recovery in a uniform medium."""
import math

import numpy as np

import workloads
from workloads.models import Spec


def _void_box(lo, hi, mesh_shape, mesh_lo=None, mesh_hi=None, sigma=(0.0, 0.0)):
    sp = Spec("mesh_box")
    root = sp.csg("root")
    box = workloads.models._box(sp, lo, hi, "vacuum")
    m = sp.mat("m", *sigma)
    sp.cell(root, box, material=m)
    sp.root = root
    sp.source = {"lo": list(lo), "hi": list(hi)}
    d = sp.to_dict()
    d["mesh"] = {"lo": list(mesh_lo or lo), "hi": list(mesh_hi or hi), "shape": list(mesh_shape)}
    return d


def _brute_ray(r, om, s, lo, hi, shape, nsamp=400000):
    """Voxel lengths of the segment r + t om, t in [0, s], by midpoint sampling of the ray."""
    lo, hi, shape = np.asarray(lo, float), np.asarray(hi, float), np.asarray(shape)
    t = (np.arange(nsamp) + 0.5) * (s / nsamp)
    p = r[None, :] + t[:, None] * om[None, :]
    ijk = np.floor((p - lo) / ((hi - lo) / shape)).astype(np.int64)
    ok = np.all((ijk >= 0) & (ijk < shape), axis=1)
    lin = ijk[ok, 0] + shape[0] * (ijk[ok, 1] + shape[1] * ijk[ok, 2])
    return np.bincount(lin, minlength=int(np.prod(shape))) * (s / nsamp)


def test_m1_axis_ray_worked_values(oracle_mod):
    """A +x ray from (0.5, 0.5, 0.5) in a void 4x2x1 box with a 4x2x1 unit mesh leaks at x = 4:
    voxel lengths 0.5, 1, 1, 1 along row (j, k) = (0, 0), nothing elsewhere."""
    spec = _void_box((0.0, 0.0, 0.0), (4.0, 2.0, 1.0), (4, 2, 1))
    m = oracle_mod.OracleModel.from_spec(spec)
    st = np.array([[0.5], [0.5], [0.5], [1.0], [0.0], [0.0]])
    res = m.run(1, states=st, mesh=True)
    want = np.zeros(8)
    want[:4] = [0.5, 1.0, 1.0, 1.0]
    assert np.array_equal(res["mesh"], want)


def test_m1_oblique_rays_match_sampling(oracle_mod):
    """Random rays through a void box with a mesh that covers part of it (voxels of unequal axes):
    per-voxel lengths equal midpoint sampling of the ray (error <= one sample spacing per plane
    crossing)."""
    lo, hi = (0.0, 0.0, 0.0), (5.0, 4.0, 3.0)
    mlo, mhi, shape = (0.5, -1.0, 0.25), (4.5, 3.5, 2.75), (5, 3, 4)
    spec = _void_box(lo, hi, shape, mlo, mhi)
    m = oracle_mod.OracleModel.from_spec(spec)
    rng = np.random.default_rng(5)
    for _ in range(20):
        r = rng.uniform(lo, hi)
        om = rng.normal(size=3)
        om /= np.linalg.norm(om)
        st = np.concatenate([r, om])[:, None]
        res = m.run(1, states=st, mesh=True, trace_cap=4)
        s = float(res["trace"]["s"][0])
        got = res["mesh"]
        want = _brute_ray(r, om, s, mlo, mhi, shape)
        nsamp = 400000
        assert np.all(np.abs(got - want) <= 2 * (s / nsamp) * 6 + 1e-12), (got, want)
        assert abs(got.sum() - want.sum()) <= 12 * s / nsamp + 1e-12


def test_m1_conservation_mesh_covers_model(oracle_mod):
    """A mesh that covers the whole C1 pincell: every segment lies inside it, so the mesh total
    equals the cell-tally total (Neumaier-summed on both sides)."""
    spec = workloads.config("c1")[0]
    hp = workloads.models.PIN_PITCH / 2
    spec["mesh"] = {"lo": [-hp, -hp, 0.0], "hi": [hp, hp, workloads.models.HEIGHT], "shape": [7, 5, 9]}
    m = oracle_mod.OracleModel.from_spec(spec)
    res = m.run(400, seed=3, mesh=True)
    assert math.isclose(res["mesh"].sum(), res["len"].sum(), rel_tol=1e-12)
    assert (res["mesh"] > 0).all()


def test_m1_voxel_volume_recovery(oracle_mod):
    """Uniform medium in an all-REFLECT box: E[mesh voxel] / E[total] = V_voxel / V_box for a mesh
    that is not aligned with anything in the model (P9 applied to the mesh)."""
    spec = workloads.models.infinite_medium(sigma_t=1.0, sigma_a=0.1)
    lo, hi = np.array(spec["source"]["lo"]), np.array(spec["source"]["hi"])
    mlo, mhi = lo + 0.1 * (hi - lo), hi - 0.3 * (hi - lo)
    shape = (3, 2, 2)
    spec["mesh"] = {"lo": mlo.tolist(), "hi": mhi.tolist(), "shape": list(shape)}
    m = oracle_mod.OracleModel.from_spec(spec)
    vfrac = np.prod((mhi - mlo) / np.array(shape)) / np.prod(hi - lo)
    B, nb = 16, 300
    fr = []
    for b in range(B):
        res = m.run(nb, seed=9, pid_begin=b * nb, mesh=True)
        fr.append(res["mesh"] / res["len"].sum())
    fr = np.array(fr)
    mean, se = fr.mean(0), fr.std(0, ddof=1) / math.sqrt(B)
    assert (np.abs(mean - vfrac) < 4.5 * se + 1e-4).all(), (mean, vfrac, se)
