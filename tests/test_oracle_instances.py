"""Oracle pins for per-instance (distributed-cell) tallies (
reading D1 in DESIGN.md): instance counts by hand, conservation against the cell tally through the
explicit depth-first enumeration, and per-instance volume recovery in a uniform medium."""
import math

import numpy as np

import workloads
from workloads.models import Spec, _box, _pin


def test_d1_instance_counts(oracle_mod):
    """Hand counts: C1 = 4 pin cells; C2 = 264 fuel pins x 4 + 25 guide tubes x 3 + 1 outer water
    pin; the instance list of C2 starts with the first fuel pin's four cells."""
    m1 = oracle_mod.OracleModel.from_spec(workloads.config("c1")[0])
    assert m1.n_instances() == 4
    m2 = oracle_mod.OracleModel.from_spec(workloads.config("c2")[0])
    assert m2.n_instances() == 264 * 4 + 25 * 3 + 1
    ic = m2.instance_cells()
    assert len(ic) == m2.n_instances()
    spec = workloads.config("c2")[0]
    fuel = next(u for u in spec["universes"] if u.get("name") == "fuel_pin")
    assert len(set(ic[:4].tolist())) == 4 == len(fuel["cells"])


def test_d1_conservation(oracle_mod):
    """Summing the instance tally over the instances of each material cell (explicit enumeration)
    gives the cell tally, for nested rect, hex and mixed models."""
    for cfg in ("c2", "c4", "c5m", "c5r"):
        m = oracle_mod.OracleModel.from_spec(workloads.config(cfg)[0])
        res = m.run(200, seed=2, instances=True)
        per_mc = np.bincount(m.instance_cells(), weights=res["inst"], minlength=m.n_mc)
        assert np.allclose(per_mc, res["len"], rtol=1e-12, atol=1e-12), cfg
        assert (res["inst"] >= 0).all()


def _uniform_lattice(sigma_t=1.0, sigma_a=0.1):
    """3x3 lattice of identical pins (fuel CZ 0.4096, water) in a reflective box, one material."""
    sp = Spec("uniform_lattice")
    root = sp.csg("root")
    p = 1.26
    box = _box(sp, (-1.5 * p, -1.5 * p, 0.0), (1.5 * p, 1.5 * p, 2.0), "reflect")
    m = sp.mat("m", sigma_t, sigma_a)
    pin = _pin(sp, "pin", (0.4096,), [m, m])
    lat = sp.rect("lat", (-1.5 * p, -1.5 * p, 0.0), (p, p, 0.0), (3, 3, 1), [pin] * 9, None)
    sp.cell(root, box, fill=lat)
    sp.root = root
    sp.source = {"lo": [-1.5 * p, -1.5 * p, 0.0], "hi": [1.5 * p, 1.5 * p, 2.0]}
    return sp.to_dict(), p


def test_d1_instance_volume_recovery(oracle_mod):
    """Uniform medium: E[L_instance] / E[L_total] = V_instance / V_box for all 18 instances
    (9 fuel discs, 9 moderator regions), in enumeration order (tile x fastest, pin cells in id
    order)."""
    spec, p = _uniform_lattice()
    m = oracle_mod.OracleModel.from_spec(spec)
    assert m.n_instances() == 18
    a_fuel = math.pi * 0.4096 ** 2
    exact = np.tile([a_fuel, p * p - a_fuel], 9) / (9 * p * p)
    B, nb = 20, 300
    fr = []
    for b in range(B):
        res = m.run(nb, seed=11, pid_begin=b * nb, instances=True)
        fr.append(res["inst"] / res["len"].sum())
    fr = np.array(fr)
    mean, se = fr.mean(0), fr.std(0, ddof=1) / math.sqrt(B)
    assert (np.abs(mean - exact) < 4.5 * se + 1e-4).all(), (mean, exact, se)
