"""Host-side checks of the C ABI (no GPU): the library loads, exports every symbol that
include/nestrack.h declares, and the builder (validation, BIH, pseudo-arrays) behaves.
No compute calls are made here (device = -1 builds are host-only)."""
import os
import re

import numpy as np
import pytest

import workloads

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def nt():
    import __graft_entry__
    from paper_2406_13849_b200 import build as nb
    nb.build()
    import paper_2406_13849_b200 as nt
    return nt


def test_exports_every_header_symbol(nt):
    hdr = open(os.path.join(ROOT, "include", "nestrack.h")).read()
    declared = sorted(set(re.findall(r"^(?:const char\*|int32_t|void|nt_status)\s+(nt_\w+)\s*\(", hdr,
                                     re.M)))
    L = nt.lib()
    missing = [s for s in declared if not hasattr(L, s)]
    assert not missing, missing
    assert set(declared) == set(nt.SYMBOLS)
    assert L.nt_abi_version() == 4


def _host(nt, spec, **kw):
    return nt.Model.from_spec(spec, device=-1, **kw)


@pytest.mark.parametrize("cfg", ["c1", "c2", "c3", "c4", "c5m", "c5r"])
def test_builder_manifest(nt, oracle_mod, cfg):
    """Material-cell bins and depth agree with the independent oracle's build."""
    spec, _ = workloads.config(cfg)
    m = _host(nt, spec)
    om = oracle_mod.OracleModel.from_spec(spec)
    assert m.info["n_material_cells"] == om.n_mc
    assert m.info["max_depth"] == om.max_depth
    assert np.array_equal(m.mc_cell, om.mc_cell)
    assert m.info["out_len"] == om.out_len


@pytest.mark.parametrize("cfg", ["c3", "c4"])
@pytest.mark.parametrize("pseudo", [False, True])
def test_bih_each_cell_exactly_once(nt, cfg, pseudo):
    """every cell of a CSG universe appears in its BIH exactly once."""
    spec, _ = workloads.config(cfg)
    m = _host(nt, spec, pseudo_array=pseudo)
    for uid, u in enumerate(spec["universes"]):
        if u["kind"] == "csg":
            info = m.bih_info(uid)
            cells = np.sort(info["leaf_cells"])
            assert len(cells) == len(set(cells.tolist())) and len(cells) == len(u["cells"])


def test_bih_deterministic_and_balanced(nt):
    spec, _ = workloads.config("c3")
    a = _host(nt, spec, pseudo_array=True)
    b = _host(nt, spec, pseudo_array=True)
    core = next(i for i, u in enumerate(spec["universes"]) if u.get("name") == "core")
    ia, ib = a.bih_info(core), b.bih_info(core)
    assert np.array_equal(ia["leaf_cells"], ib["leaf_cells"]) and ia["n_nodes"] == ib["n_nodes"]
    n = len(ia["leaf_cells"])
    assert n > 300                       # 19 x 19 pseudo tiles
    assert ia["depth"] <= 3 * int(np.ceil(np.log2(n)))


def _tiny():
    sp = workloads.models.Spec("tiny")
    root = sp.csg("root")
    box = workloads.models._box(sp, (-1, -1, -1), (1, 1, 1), "vacuum")
    m = sp.mat("m", 1.0, 0.5)
    sp.cell(root, box, material=m)
    sp.root = root
    sp.source = {"lo": [-1, -1, -1], "hi": [1, 1, 1]}
    return sp


@pytest.mark.parametrize("mutate,needle", [
    (lambda d: d["materials"][0].update(sigma_a=2.0), "sigma_a"),
    (lambda d: d["surfaces"].append({"kind": "CZ", "coef": [0, 0, -1.0], "bc": "none"}), "radius"),
    (lambda d: d["surfaces"].append({"kind": "CZ", "coef": [0, 0, 1.0], "bc": "reflect"}), "REFLECT"),
    (lambda d: d["universes"][0]["cells"][0]["hs"].append(1), "twice"),
    (lambda d: d["universes"][0]["cells"][0]["hs"].append(99), "out of range"),
])
def test_invalid_models_rejected(nt, mutate, needle):
    d = _tiny().to_dict()
    mutate(d)
    with pytest.raises(nt.NtError) as e:
        _host(nt, d)
    assert e.value.status == -4 and needle in str(e.value)


def test_cycle_and_bc_scope_rejected(nt):
    sp = _tiny()
    u = sp.csg("inner")
    m = 0
    sp.cell(u, [], fill=0)                      # inner -> root: a cycle once root -> inner
    sp.universes[0]["cells"][0] = {"hs": sp.universes[0]["cells"][0]["hs"], "fill": u}
    with pytest.raises(nt.NtError, match="cycle"):
        _host(nt, sp.to_dict())
    sp2 = _tiny()
    v = sp2.csg("inner")
    s = sp2.surf("CZ", [0, 0, 0.5], "vacuum")
    sp2.cell(v, [-(s + 1)], material=0)
    sp2.cell(v, [s + 1], material=0)
    sp2.universes[0]["cells"][0] = {"hs": sp2.universes[0]["cells"][0]["hs"], "fill": v}
    with pytest.raises(nt.NtError, match="boundary condition"):
        _host(nt, sp2.to_dict())


def test_order_errors(nt):
    m = nt.Model()
    with pytest.raises(nt.NtError) as e:
        m.make_run(1, 1)
        import ctypes as C
        st = nt.lib().nt_track(m.h, C.byref(m.make_run(1, 1)), C.byref(nt.Outputs()), None)
        nt._check(st)
    spec = _tiny().to_dict()
    m = _host(nt, spec)
    with pytest.raises(nt.NtError) as e:
        m.add_material(1.0, 0.1)
    assert e.value.status == -3


def test_track_on_host_only_model_is_an_error(nt):
    import ctypes as C
    m = _host(nt, _tiny().to_dict())
    o = nt.Outputs()
    buf = np.zeros(64)
    o.out = buf.ctypes.data
    st = nt.lib().nt_track(m.h, C.byref(m.make_run(10, 1)), C.byref(o), None)
    assert st == -3


def test_pseudo_array_cell_counts(nt):
    spec, _ = workloads.config("c2")
    a = _host(nt, spec)
    b = _host(nt, spec, pseudo_array=True)
    assert b.info["n_cells"] - a.info["n_cells"] >= 19 * 19    # 17x17 + rings of outer tiles
    assert b.info["n_material_cells"] == a.info["n_material_cells"]
    spec4, _ = workloads.config("c4")
    c = _host(nt, spec4, pseudo_array=True)
    assert c.info["n_cells"] > 217 + 19


@pytest.mark.parametrize("cfg,ok,K", [("c1", 1, 0), ("c2", 1, 1), ("c3", 1, 2), ("c5r", 1, 3),
                                      ("c4", 0, 0), ("c5m", 0, 0)])
def test_rect_specialisable_gate(nt, cfg, ok, K):
    """NT_TRACKER_RECT accepts exactly the root -> RECT^K -> pin models (Alg. 9-10 shape)."""
    spec, _ = workloads.config(cfg)
    m = _host(nt, spec)
    assert m.info["rect_specialisable"] == ok
    if ok:
        assert m.info["rect_levels"] == K


def test_nonuniform_rect_host_build(nt):
    """Non-uniform rect arrays (Alg. 5, reading N1): build, feature bit, rect-tracker gate,
    pseudo-array conversion (every tile -1..n per axis), edge validation."""
    spec = workloads.models.nonuniform_slabs()
    m = _host(nt, spec)
    assert m.info["rect_specialisable"] == 0
    assert m.info["max_depth"] == 3
    p = _host(nt, spec, pseudo_array=True)
    assert p.info["n_cells"] == 1 + 12 + 12            # root box + tiles (+ their all-space cells)
    g = _host(nt, workloads.models.gap_lattice(True), pseudo_array=True)
    assert g.info["n_cells"] > 7 * 7
    bad = workloads.models.nonuniform_slabs()
    lat = next(u for u in bad["universes"] if u["kind"] == "rect")
    lat["edges"][0] = [0.0, 3.0, 1.0, 6.0]
    with pytest.raises(nt.NtError, match="strictly increasing"):
        _host(nt, bad)


def test_mesh_host_validation(nt):
    """nt_set_mesh (NEXT-2): voxel count reported by nt_model_info; bad shapes / boxes rejected."""
    spec, _ = workloads.config("c3")
    spec["mesh"] = {"lo": [-161.25, -161.25, 0.0], "hi": [161.25, 161.25, 365.76], "shape": [119, 119, 30]}
    m = _host(nt, spec)
    assert m.info["mesh_bins"] == 119 * 119 * 30
    assert _host(nt, workloads.config("c1")[0]).info["mesh_bins"] == 0
    for bad in ({"shape": [0, 1, 1]}, {"hi": [-161.25, 161.25, 365.76]}):
        s2 = dict(spec)
        s2["mesh"] = dict(spec["mesh"], **bad)
        with pytest.raises(nt.NtError, match="nt_set_mesh"):
            _host(nt, s2)


def test_instance_tables_host(nt, oracle_mod):
    """D1 instance numbering: the builder's enumeration equals the oracle's (independent DFS),
    and pseudo-array builds report no instances."""
    for cfg in ("c1", "c2", "c4", "c5m", "c5r"):
        spec, _ = workloads.config(cfg)
        m = _host(nt, spec)
        om = oracle_mod.OracleModel.from_spec(spec)
        assert m.info["n_instances"] == om.n_instances()
        assert np.array_equal(m.instance_cells(), om.instance_cells())
    assert _host(nt, workloads.config("c2")[0], pseudo_array=True).info["n_instances"] == 0


def test_fission_host_validation(nt):
    """nt_set_fission (F1): max_sites in the model info; a fissile material without absorption is
    rejected at nt_finalize."""
    spec = workloads.models.with_fission(workloads.config("c1")[0], {"uo2": 0.15})
    m = _host(nt, spec)
    assert m.info["max_sites"] == int(np.floor(0.15 / 0.12)) + 1
    assert _host(nt, workloads.config("c1")[0]).info["max_sites"] == 1
    bad = workloads.models.with_fission(workloads.config("c1")[0], {"gap": 0.1})   # sigma_a = 0
    with pytest.raises(nt.NtError, match="nu_sigma_f"):
        _host(nt, bad)
