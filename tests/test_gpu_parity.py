"""GPU parity: the CUDA path (through the C ABI) against the independent CPU oracle.

Contract (BASELINE.json north_star): event/cell/surface sequences
bit-exact; segment lengths within 1e-12 relative (the build reaches bit-identity because both
sides follow the same spec'd arithmetic); per-cell totals within 1e-9 relative (summation order);
counters exact.  Flagged histories (O16) would be excluded, but with bit-identical walks none
needs to be.
"""
import numpy as np
import pytest

import workloads

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TRACE_FIELDS = ("pid", "seg", "kind", "level", "j", "cell_before", "cell_after", "terminal", "flags")


@pytest.fixture(scope="module")
def nt():
    import __graft_entry__
    __graft_entry__.build()
    import paper_2406_13849_b200 as nt
    assert torch.cuda.is_available()
    return nt


@pytest.fixture(scope="module")
def orc():
    import oracle
    oracle.build()
    return oracle


def _compare(nt, orc, spec, n, seed, pid_begin=0, max_segments=0, states=None, tracker="generic",
             trace=True, pseudo=False, scheduler="block", block_dim=0):
    m = nt.Model.from_spec(spec, device=0, pseudo_array=pseudo)
    om = orc.OracleModel.from_spec(spec)
    cap = 400 * max(n, 1) + 64 if trace else 0
    st_t = None if states is None else torch.tensor(states, dtype=torch.float64, device="cuda")
    res = m.track(n, seed=seed, pid_begin=pid_begin, pflags=True, per_history=True, trace_cap=cap,
                  max_segments=max_segments, states=st_t, tracker=tracker, scheduler=scheduler,
                  block_dim=block_dim)
    torch.cuda.synchronize()
    g = m.unpack(res["out"])
    o = om.run(n, seed=seed, pid_begin=pid_begin, pflags=True, trace_cap=cap, max_segments=max_segments,
               states=states, per_history=True)
    assert g["counters"] == o["counters"]
    assert np.array_equal(g["exits"], o["exits"])
    assert np.allclose(g["len"], o["len"], rtol=1e-12, atol=1e-300)
    assert np.array_equal(res["pflags"].cpu().numpy()[:n], o["pflags"])
    if trace:
        gt, ot = nt.Model.trace_records(res), o["trace"]
        assert len(gt) == len(ot)
        for f in TRACE_FIELDS:
            assert np.array_equal(gt[f], ot[f]), f
        # per-segment tolerance of the contract, then the stronger bit-identity we reach
        assert np.all(np.abs(gt["s"] - ot["s"]) <= 1e-12 * np.abs(ot["s"]) + 1e-13)
        assert np.array_equal(gt["s"], ot["s"])
    # per-history segment counts and terminals equal the oracle's, history by history
    nseg = res["pnseg"].cpu().numpy()[:n]
    assert np.array_equal(nseg, o["pnseg"].astype(np.int32))
    assert np.array_equal(res["pterm"].cpu().numpy()[:n], o["pterm"])
    assert nseg.sum() == g["counters"]["segments"]
    return m, g, o, res


# the rect-specialised tracker: history-based ("rect") and on the ring event queues ("rect-ring")
RECT_KW = {"rect": dict(tracker="rect", scheduler="history"), "rect-ring": dict(tracker="rect", scheduler="block")}

CONFIG_N = {"c1": 2000, "c2": 600, "c3": 600, "c4": 600, "c5m": 600, "c5r": 600}


@pytest.mark.parametrize("sched", ["warp", "block", "history", "dp", "rounds", "dp-rounds"])
@pytest.mark.parametrize("cfg", list(CONFIG_N))
def test_config_trace_parity(nt, orc, cfg, sched):
    """Every BASELINE config: full traces bit-exact vs the oracle (seeded, small batch), with
    both schedulers (event queues / history-based)."""
    spec, _ = workloads.config(cfg)
    _, g, o, _ = _compare(nt, orc, spec, CONFIG_N[cfg], seed=1, scheduler=sched)
    assert g["counters"]["lost"] == 0 and g["counters"]["capped"] == 0


@pytest.mark.parametrize("cfg", ["c3", "c4", "c5m"])
def test_config_trace_parity_block192(nt, orc, cfg):
    """Ring-queue scheduler with 192-slot blocks (6 warps, more blocks per SM): traces bit-exact."""
    spec, _ = workloads.config(cfg)
    _compare(nt, orc, spec, CONFIG_N[cfg], seed=1, block_dim=192)


@pytest.mark.parametrize("seed", workloads.PARITY_SEEDS)
def test_c3_parity_seeds(nt, orc, seed):
    spec, _ = workloads.config("c3")
    _compare(nt, orc, spec, 1000, seed=seed, pid_begin=12345, trace=False)


@pytest.mark.parametrize("cfg", ["c1", "c2", "c4"])
def test_config_parity_untraced(nt, orc, cfg):
    """Untraced runs take the ring scheduler's 320-slot kernel where it fits (a traced run needs more
    shared memory per slot and keeps 256): counters, exits, lengths and flags against the oracle."""
    spec, _ = workloads.config(cfg)
    _compare(nt, orc, spec, 3000, seed=2, pid_begin=777, trace=False)


@pytest.mark.parametrize("name", ["sphere_in_box", "hex_pins_small_pointy", "hex_pins_small_flat",
                                  "rect3d_small", "lattice3_nested", "lattice3_flat", "infinite_medium",
                                  "c1_void_vacuum", "slab_mix"])
@pytest.mark.parametrize("sched", ["block", "dp", "rounds"])
def test_test_models_parity(nt, orc, name, sched):
    """Planes, spheres, 3-D rect and hex z-stacks, translations, void + vacuum leakage."""
    M = workloads.models
    spec = {"sphere_in_box": M.sphere_in_box, "hex_pins_small_pointy": lambda: M.hex_pins_small("pointy"),
            "hex_pins_small_flat": lambda: M.hex_pins_small("flat"), "rect3d_small": M.rect3d_small,
            "lattice3_nested": M.lattice3_nested, "lattice3_flat": lambda: M.lattice3_nested(True),
            "infinite_medium": M.infinite_medium,
            "c1_void_vacuum": lambda: M.c1_pincell(bc="vacuum", void=True), "slab_mix": M.slab_mix}[name]()
    _compare(nt, orc, spec, 700, seed=2, scheduler=sched)


NONUNIFORM = {"gap_lattice": lambda: workloads.models.gap_lattice(True),
              "c2_gap_assembly": lambda: workloads.models.c2_gap_assembly(),
              "nonuniform_slabs": lambda: workloads.models.nonuniform_slabs()}


@pytest.mark.parametrize("sched", ["block", "warp", "history", "dp", "rounds"])
@pytest.mark.parametrize("name", list(NONUNIFORM))
def test_nonuniform_rect_parity(nt, orc, name, sched):
    """Non-uniform rect arrays (Alg. 5 binary search, reading N1): traces bit-exact vs the oracle
    under every scheduler / dispatch."""
    _compare(nt, orc, NONUNIFORM[name](), 600, seed=8, scheduler=sched)


@pytest.mark.parametrize("name", ["gap_lattice", "c2_gap_assembly"])
def test_nonuniform_pseudo_array_equals_generic(nt, name):
    """ST conversion of a non-uniform array (planes at the divisions, slabs -1 / n bounded on one
    side): same walk as the binary-search lattice (surface ids j differ by construction)."""
    spec = NONUNIFORM[name]()
    a = nt.Model.from_spec(spec, device=0)
    b = nt.Model.from_spec(spec, device=0, pseudo_array=True)
    ra = a.track(600, seed=7, trace_cap=400000, pflags=True)
    rb = b.track(600, seed=7, trace_cap=400000, pflags=True)
    torch.cuda.synchronize()
    ta, tb = nt.Model.trace_records(ra), nt.Model.trace_records(rb)
    assert len(ta) == len(tb)
    for f in ("pid", "seg", "kind", "level", "cell_before", "cell_after", "terminal", "s"):
        assert np.array_equal(ta[f], tb[f]), f


def _with_mesh(spec, lo, hi, shape):
    spec = dict(spec)
    spec["mesh"] = {"lo": list(lo), "hi": list(hi), "shape": list(shape)}
    return spec


MESHED = {
    # C1 pincell, mesh over the whole box (every segment scored)
    "c1": lambda: _with_mesh(workloads.config("c1")[0], (-0.63, -0.63, 0.0), (0.63, 0.63, 365.76), (7, 5, 9)),
    # C3 core with a coarse mesh over part of the core (segments cross in and out of it)
    "c3": lambda: _with_mesh(workloads.config("c3")[0], (-120.0, -161.25, 20.0), (161.25, 100.0, 300.0), (23, 19, 7)),
    # C4 hex core, mesh larger than the model
    "c4": lambda: _with_mesh(workloads.config("c4")[0], (-120.0, -120.0, -10.0), (120.0, 120.0, 160.0), (16, 16, 4)),
}


@pytest.mark.parametrize("sched", ["block", "warp", "history", "dp", "rounds", "rect", "rect-ring"])
@pytest.mark.parametrize("name", list(MESHED))
def test_mesh_tally_parity(nt, orc, name, sched):
    """Superimposed mesh track-length tally (NEXT-2, reading M1): per-voxel totals vs the oracle's
    sort-the-cuts definition, within 1e-9 relative (summation order), under every scheduler."""
    spec = MESHED[name]()
    m = nt.Model.from_spec(spec, device=0)
    if sched.startswith("rect") and not m.info["rect_specialisable"]:
        pytest.skip("not rect-specialisable")
    om = orc.OracleModel.from_spec(spec)
    n = 400
    kw = RECT_KW.get(sched, dict(scheduler=sched))
    res = m.track(n, seed=4, mesh=True, **kw)
    torch.cuda.synchronize()
    o = om.run(n, seed=4, mesh=True)
    g = m.unpack(res["out"])
    assert g["counters"] == o["counters"]
    gm, ref = res["mesh"].cpu().numpy(), o["mesh"]
    assert gm.shape == ref.shape and (ref > 0).sum() > 10
    assert np.all(np.abs(gm - ref) <= 1e-9 * np.abs(ref) + 1e-12 * ref.max())
    if name == "c1":                                  # mesh covers the model: conservation
        assert np.isclose(gm.sum(), g["len"].sum(), rtol=1e-12)


def test_mesh_tally_off_without_buffer(nt):
    """A model with a mesh run without outputs.mesh: cell tallies only, identical to no mesh."""
    spec = MESHED["c1"]()
    a = nt.Model.from_spec(spec, device=0)
    b = nt.Model.from_spec(workloads.config("c1")[0], device=0)
    ra, rb = a.track(500, seed=2), b.track(500, seed=2)
    torch.cuda.synchronize()
    assert torch.equal(ra["out"], rb["out"]) or np.allclose(ra["out"].cpu().numpy(), rb["out"].cpu().numpy(), rtol=1e-13)


@pytest.mark.parametrize("sched", ["block", "rounds", "warp", "history", "dp"])
@pytest.mark.parametrize("cfg", ["c2", "c4", "c5m"])
def test_instance_tally_parity(nt, orc, cfg, sched):
    """Per-instance (distributed-cell) tally, reading D1: every instance's track length vs the
    oracle (which numbers instances by summing earlier siblings' leaves level by level)."""
    spec, _ = workloads.config(cfg)
    m = nt.Model.from_spec(spec, device=0)
    om = orc.OracleModel.from_spec(spec)
    n = 400
    res = m.track(n, seed=6, instances=True, scheduler=sched)
    torch.cuda.synchronize()
    o = om.run(n, seed=6, instances=True)
    gi = res["inst"].cpu().numpy()[:om.n_instances()]
    ref = o["inst"]
    assert (ref > 0).sum() > 20
    assert np.all(np.abs(gi - ref) <= 1e-9 * np.abs(ref) + 1e-12 * ref.max())


@pytest.mark.parametrize("name", ["nonuniform_slabs", "gap_lattice", "hex_pins_small_flat", "rect3d_small"])
def test_instance_tally_test_models(nt, orc, name):
    """Instance numbering through non-uniform rect, 3-D rect and hex arrays (with outer tiles)."""
    M = workloads.models
    spec = {"nonuniform_slabs": M.nonuniform_slabs, "gap_lattice": lambda: M.gap_lattice(True),
            "hex_pins_small_flat": lambda: M.hex_pins_small("flat"), "rect3d_small": M.rect3d_small}[name]()
    m = nt.Model.from_spec(spec, device=0)
    om = orc.OracleModel.from_spec(spec)
    assert np.array_equal(m.instance_cells(), om.instance_cells())
    res = m.track(500, seed=13, instances=True)
    torch.cuda.synchronize()
    o = om.run(500, seed=13, instances=True)
    gi, ref = res["inst"].cpu().numpy()[:om.n_instances()], o["inst"]
    assert np.all(np.abs(gi - ref) <= 1e-9 * np.abs(ref) + 1e-12 * ref.max())


def test_mesh_and_instance_tallies_together(nt, orc):
    """Both extra tallies in one run (separate kernel instantiation) on the full-core model."""
    spec = MESHED["c3"]()
    m = nt.Model.from_spec(spec, device=0)
    om = orc.OracleModel.from_spec(spec)
    res = m.track(300, seed=9, mesh=True, instances=True)
    torch.cuda.synchronize()
    o = om.run(300, seed=9, mesh=True, instances=True)
    g = m.unpack(res["out"])
    assert g["counters"] == o["counters"]
    for key in ("mesh", "inst"):
        got, ref = res[key].cpu().numpy()[:len(o[key])], o[key]
        assert np.all(np.abs(got - ref) <= 1e-9 * np.abs(ref) + 1e-12 * ref.max()), key


FISSILE = {
    "c1": lambda: workloads.models.with_fission(workloads.config("c1")[0], {"uo2": 0.15}),
    "c3": lambda: workloads.models.with_fission(workloads.config("c3")[0],
                                                 {"uo2_a": 0.13, "uo2_b": 0.16, "uo2_c": 0.19}),
}


@pytest.mark.parametrize("sched", ["block", "rounds", "warp", "history", "dp", "rect", "rect-ring"])
@pytest.mark.parametrize("cfg", list(FISSILE))
def test_fission_bank_parity(nt, orc, cfg, sched):
    """F1 fission bank: sites per history and site coordinates bit-exact vs the oracle."""
    spec = FISSILE[cfg]()
    m = nt.Model.from_spec(spec, device=0)
    om = orc.OracleModel.from_spec(spec)
    assert m.info["max_sites"] == om.max_sites()
    n = 700
    kw = RECT_KW.get(sched, dict(scheduler=sched))
    res = m.track(n, seed=12, bank=True, **kw)
    torch.cuda.synchronize()
    o = om.run(n, seed=12, bank=True)
    bn = res["bank_n"].cpu().numpy()[:n]
    assert np.array_equal(bn, o["bank_n"]) and bn.sum() > 50
    bk = res["bank"].cpu().numpy()[:n * om.max_sites() * 3].reshape(n, om.max_sites(), 3)
    for h in np.nonzero(bn)[0]:
        assert np.array_equal(bk[h, :bn[h]], o["bank"][h, :bn[h]])


def test_fission_source_and_power_iteration_parity(nt, orc):
    """F1 source resampling on the device = the oracle's (bit-exact states), and three power
    iteration cycles give the oracle's k sequence exactly."""
    spec = FISSILE["c1"]()
    m = nt.Model.from_spec(spec, device=0)
    om = orc.OracleModel.from_spec(spec)
    n = 1500
    res = m.track(n, seed=3, bank=True)
    torch.cuda.synchronize()
    st, M = m.fission_source(res["bank"], res["bank_n"], n, seed=3, cycle=0, n_next=1200)
    torch.cuda.synchronize()
    ms = om.max_sites()
    bank = res["bank"].cpu().numpy()[:n * ms * 3].reshape(n, ms, 3)
    bank_n = res["bank_n"].cpu().numpy()[:n]
    ost, oM = om.fission_source(np.where(np.arange(ms)[None, :, None] < bank_n[:, None, None], bank, 0.0),
                                bank_n, seed=3, cycle=0, n_next=1200)
    assert M == oM == int(bank_n.sum())
    assert np.array_equal(st.cpu().numpy(), ost)
    assert m.power_iteration(n, cycles=3, seed=5) == om.power_iteration(n, cycles=3, seed=5)


def test_fission_k_inf_on_device(nt):
    """Infinite medium with fission: the device's k estimates k_inf = nu Sigma_f / Sigma_a."""
    spec = workloads.infinite_medium(1.0, 0.25, 0.55)
    m = nt.Model.from_spec(spec, device=0)
    ks = m.power_iteration(200000, cycles=3, seed=9)
    nut, p = 2.2, 0.2
    assert abs(np.mean(ks) - nut) < 4.5 * np.sqrt(p * (1 - p) / (3 * 200000))


def test_dp_dispatch_rejects_other_schedulers(nt):
    """NT_DP is a dispatch mode of the block-queue scheduler only (nestrack.h)."""
    spec, _ = workloads.config("c1")
    m = nt.Model.from_spec(spec, device=0)
    for kw in ({"block_dim": 128}, {"tracker": "rect"}):
        with pytest.raises(nt.NtError):
            m.track(10, seed=1, scheduler="dp", **kw)
    run = m.make_run(10, 1, scheduler="history")
    run.flags |= nt.NT_DP
    out = torch.zeros(m.out_len, dtype=torch.float64, device="cuda")
    o = nt.Outputs()
    o.out = out.data_ptr()
    assert m.L.nt_track(m.h, nt.C.byref(run), nt.C.byref(o), None) == -1


@pytest.mark.parametrize("block", [128, 192, 256])
@pytest.mark.parametrize("n", [1, 31, 257, 1000])
def test_ragged_batches_and_large_pids(nt, orc, n, block):
    """Ragged batch sizes (partial warps / blocks) and pids above 2^32 (counter hi word)."""
    spec, _ = workloads.config("c2")
    _compare(nt, orc, spec, n, seed=3, pid_begin=(1 << 33) + 17, block_dim=block, scheduler="block")
    _compare(nt, orc, spec, n, seed=3, pid_begin=(1 << 33) + 17, scheduler="warp")


@pytest.mark.parametrize("sched", ["warp", "block", "history", "dp", "rounds"])
def test_capped_histories(nt, orc, sched):
    """max_segments reached -> CAPPED (F3) on both sides, same extra trace record."""
    spec, _ = workloads.config("c1")
    _, g, o, _ = _compare(nt, orc, spec, 300, seed=4, max_segments=7, scheduler=sched)
    assert g["counters"]["capped"] > 0


@pytest.mark.parametrize("sched", ["warp", "block", "history", "dp", "rounds"])
def test_lost_at_birth(nt, orc, sched):
    """Births outside every root cell are LOST at birth (source box larger than the model)."""
    spec = workloads.c1_pincell()
    spec["source"] = {"lo": [-1.0, -1.0, 0.0], "hi": [1.0, 1.0, 365.76]}
    _, g, o, _ = _compare(nt, orc, spec, 500, seed=5, scheduler=sched)
    assert g["counters"]["lost"] > 0


@pytest.mark.parametrize("sched", ["warp", "block", "history", "dp", "rounds"])
def test_explicit_states(nt, orc, sched):
    """nt_track_states: explicit birth states (chord rays through the void pincell)."""
    spec = workloads.c1_pincell(bc="vacuum", void=True)
    rng = np.random.default_rng(0)
    n = 500
    r = rng.uniform([-0.63, -0.63, 0.0], [0.63, 0.63, 365.76], size=(n, 3))
    om = rng.normal(size=(n, 3))
    om /= np.linalg.norm(om, axis=1, keepdims=True)
    _compare(nt, orc, spec, n, seed=6, states=np.concatenate([r.T, om.T]), scheduler=sched)


def test_zero_particles(nt):
    spec, _ = workloads.config("c1")
    m = nt.Model.from_spec(spec, device=0)
    res = m.track(0, seed=1)
    torch.cuda.synchronize()
    assert float(res["out"].abs().sum()) == 0.0


def test_find_cells_parity(nt, orc):
    """Point location (Alg. 7) on random points of every config, exact cell ids."""
    rng = np.random.default_rng(1)
    for cfg in CONFIG_N:
        spec, _ = workloads.config(cfg)
        m = nt.Model.from_spec(spec, device=0)
        om = orc.OracleModel.from_spec(spec)
        lo, hi = np.array(spec["source"]["lo"]), np.array(spec["source"]["hi"])
        pts = rng.uniform(lo, hi, size=(20000, 3)).T.copy()
        gc, gf = m.find_cells(torch.tensor(pts, device="cuda"))
        oc, of = om.find_cells(pts)
        assert np.array_equal(gc.cpu().numpy(), oc)
        assert np.array_equal(gf.cpu().numpy(), of)


@pytest.mark.parametrize("cfg", ["c2", "c3", "c5r"])
def test_pseudo_array_equals_generic(nt, cfg):
    """P13: pseudo-array (ST) mode = generic tracker for RECT lattices: same walk, bit-exact
    (surface ids j differ by construction)."""
    spec, _ = workloads.config(cfg)
    a = nt.Model.from_spec(spec, device=0)
    b = nt.Model.from_spec(spec, device=0, pseudo_array=True)
    ra = a.track(600, seed=7, trace_cap=400000, pflags=True)
    rb = b.track(600, seed=7, trace_cap=400000, pflags=True)
    torch.cuda.synchronize()
    ta, tb = nt.Model.trace_records(ra), nt.Model.trace_records(rb)
    ok = (ra["pflags"] == 0) & (rb["pflags"] == 0)
    ok = ok.cpu().numpy()[:600]
    ma, mb = ok[(ta["pid"]).astype(np.int64)], ok[(tb["pid"]).astype(np.int64)]
    ta, tb = ta[ma], tb[mb]
    assert len(ta) == len(tb)
    for f in ("pid", "seg", "kind", "level", "cell_before", "cell_after", "terminal", "s"):
        assert np.array_equal(ta[f], tb[f]), f


@pytest.mark.parametrize("cfg", ["c4", "c5m"])
def test_pseudo_hex_locates_same_cells(nt, cfg):
    """ST mode on HEX lattices (hexagonal prisms of general planes, polytope AABBs): point
    location gives the same material cell as the closed-form hex indexing.  Hex tiles are plane
    cells here, so points within rounding of a tile edge may legitimately differ."""
    spec, _ = workloads.config(cfg)
    a = nt.Model.from_spec(spec, device=0)
    b = nt.Model.from_spec(spec, device=0, pseudo_array=True)
    rng = np.random.default_rng(3)
    lo, hi = np.array(spec["source"]["lo"]), np.array(spec["source"]["hi"])
    pts = torch.tensor(rng.uniform(lo, hi, size=(200000, 3)).T.copy(), device="cuda")
    ca, fa = a.find_cells(pts)
    cb, fb = b.find_cells(pts)
    assert int((fb != 0).sum()) == int((fa != 0).sum())
    assert int((ca != cb).sum()) <= 2


def test_host_entry_point(nt):
    """nt_track_host (host output buffer) equals the device-buffer call."""
    spec, _ = workloads.config("c2")
    m = nt.Model.from_spec(spec, device=0)
    a = m.track(5000, seed=9)["out"].cpu().numpy()
    b = m.track_host(5000, seed=9)
    assert np.array_equal(a[-18:], b[-18:])
    assert np.allclose(a, b, rtol=1e-12, atol=0)


def test_determinism_and_additivity(nt):
    """Counters exact and lengths to summation order across repeat runs and pid splits (P14)."""
    spec, _ = workloads.config("c3")
    m = nt.Model.from_spec(spec, device=0)
    ab = m.unpack(m.track(200000, seed=11)["out"])
    ab2 = m.unpack(m.track(200000, seed=11)["out"])
    a = m.unpack(m.track(70000, seed=11)["out"])
    b = m.unpack(m.track(130000, seed=11, pid_begin=70000)["out"])
    assert ab["counters"] == ab2["counters"]
    assert ab["counters"] == {k: a["counters"][k] + b["counters"][k] for k in ab["counters"]}
    assert np.allclose(ab["len"], a["len"] + b["len"], rtol=1e-11, atol=0)
    assert np.allclose(ab["len"], ab2["len"], rtol=1e-11, atol=0)


def test_full_size_c3_sampled(nt, orc):
    """BASELINE size (C3, 1e8 histories) in the bench launch configuration: invariants on the
    whole batch, and per-history segment counts / terminals / flags of sampled pid windows
    recomputed one by one by the oracle."""
    spec, n = workloads.config("c3")
    m = nt.Model.from_spec(spec, device=0)
    res = m.track(n, seed=workloads.SEED, pflags=True, per_history=True)
    torch.cuda.synchronize()
    g = m.unpack(res["out"])
    c = g["counters"]
    assert c["particles"] == n and c["lost"] == 0 and c["capped"] == 0
    assert c["segments"] == c["crossings"] + c["reflections"] + c["collisions"]
    assert c["particles"] == c["absorptions"] + c["leaks"]
    assert int(res["pnseg"].sum()) == c["segments"]
    om = orc.OracleModel.from_spec(spec)
    nseg = res["pnseg"]
    term = res["pterm"]
    fl = res["pflags"]
    rng = np.random.default_rng(2)
    starts = sorted(set([0, n - 64] + list(rng.integers(0, n - 64, size=14))))
    for s0 in starts:
        o = om.run(64, seed=workloads.SEED, pid_begin=int(s0), pflags=True, trace_cap=64 * 400)
        per = np.bincount(o["trace"]["pid"].astype(np.int64) - int(s0), minlength=64)
        assert np.array_equal(nseg[s0:s0 + 64].cpu().numpy(), per)
        assert np.array_equal(fl[s0:s0 + 64].cpu().numpy(), o["pflags"])
        last = o["trace"][np.r_[np.nonzero(np.diff(o["trace"]["pid"]))[0], len(o["trace"]) - 1]]
        assert np.array_equal(term[s0:s0 + 64].cpu().numpy(), last["terminal"])


@pytest.mark.parametrize("cfg", ["c1", "c2", "c3", "c5r"])
@pytest.mark.parametrize("sched", ["history", "block"])
def test_rect_tracker_bit_identical(nt, orc, cfg, sched):
    """P13: the rect-specialised tracker (Alg. 9-10 analogue), history-based and on the ring event
    queues, reproduces the generic tracker and the oracle bit for bit on every rect-shaped config."""
    spec, _ = workloads.config(cfg)
    _compare(nt, orc, spec, 600, seed=8, tracker="rect", scheduler=sched)
    _compare(nt, orc, spec, 40, seed=9, tracker="rect", scheduler=sched, max_segments=25)


def test_rect_tracker_full_counters_match_generic(nt):
    spec, _ = workloads.config("c3")
    m = nt.Model.from_spec(spec, device=0)
    a = m.unpack(m.track(300000, seed=13)["out"])
    for sched in ("history", "block"):
        b = m.unpack(m.track(300000, seed=13, tracker="rect", scheduler=sched)["out"])
        assert a["counters"] == b["counters"]
        assert np.array_equal(a["exits"], b["exits"])
        assert np.allclose(a["len"], b["len"], rtol=1e-11, atol=0)


@pytest.mark.parametrize("cfg", ["c4", "c5m"])
def test_rect_tracker_rejects_hex(nt, cfg):
    spec, _ = workloads.config(cfg)
    m = nt.Model.from_spec(spec, device=0)
    with pytest.raises(nt.NtError) as e:
        m.track(10, seed=1, tracker="rect")
    assert e.value.status == -5


def test_fast_division_sqrt_are_ieee(nt):
    """The kernels' slow-path-free division / sqrt return the IEEE results bit for bit on 2^26
    random operands spanning (and exceeding) the walk's ranges."""
    assert nt.selftest_arith(1 << 26, 3) == (0, 0)


def test_power_iteration_distributed_single_rank(nt, orc):
    """The multi-GPU driver's device path (nt_bank_compact + nt_source_from_sites) at one rank
    equals the single-GPU power iteration and the oracle's, cycle by cycle."""
    spec = FISSILE["c1"]()
    m = nt.Model.from_spec(spec, device=0)
    om = orc.OracleModel.from_spec(spec)
    ks = nt.power_iteration_distributed(m, 1000, 3, seed=8)
    assert ks == m.power_iteration(1000, cycles=3, seed=8) == om.power_iteration(1000, cycles=3, seed=8)


_SLOTS_SCRIPT = r"""
import sys, json, hashlib
sys.path.insert(0, sys.argv[1])
import torch, workloads, paper_2406_13849_b200 as nt
m = nt.Model.from_spec(workloads.c3_full_core(), device=0)
res = m.track(200000, seed=5, pid_begin=123456, pflags=True, per_history=True)
torch.cuda.synchronize()
g = m.unpack(res["out"])
h = hashlib.sha256()
for k in ("pflags", "pnseg", "pterm"):
    h.update(res[k].cpu().numpy().tobytes())
print(json.dumps({"counters": g["counters"], "exits": [int(x) for x in g["exits"]],
                  "len": [float(x).hex() for x in g["len"]], "per_history": h.hexdigest()}))
"""


def test_ring_slot_counts_agree(nt):
    """The ring scheduler's 320-slot and 256-slot kernels (NESTRACK_SLOTS, read once per process)
    give the same walks: counters, exits and every history's segment count, terminal and flags
    equal; lengths to summation order."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = {}
    for slots in ("256", "320"):
        env = dict(os.environ, NESTRACK_SLOTS=slots)
        p = subprocess.run([sys.executable, "-c", _SLOTS_SCRIPT, root], env=env, capture_output=True, text=True,
                           timeout=600)
        assert p.returncode == 0, p.stderr[-2000:]
        outs[slots] = json.loads(p.stdout.strip().splitlines()[-1])
    a, b = outs["256"], outs["320"]
    assert a["counters"] == b["counters"] and a["exits"] == b["exits"]
    assert a["per_history"] == b["per_history"]
    la = np.array([float.fromhex(x) for x in a["len"]])
    lb = np.array([float.fromhex(x) for x in b["len"]])
    assert np.allclose(la, lb, rtol=1e-12, atol=0)


@pytest.mark.parametrize("cfg", ["c4", "c5m"])
def test_fh_kernel_equals_f7(nt, cfg, monkeypatch):
    """Hex + general-plane models run the default path in the fh feature set (track_fh.cu, a smaller
    kernel); NESTRACK_NO_FH=1 forces the f7 kernels.  Both must give identical walks: exact counters,
    exits, per-history segment counts and terminals, bit-identical track-length totals."""
    spec, _ = workloads.config(cfg)
    m = nt.Model.from_spec(spec, device=0)
    n = 300000   # >> resident slots: slots are recycled
    outs = []
    for off in (False, True):
        if off:
            monkeypatch.setenv("NESTRACK_NO_FH", "1")
        res = m.track(n, seed=17, per_history=True)
        torch.cuda.synchronize()
        outs.append((m.unpack(res["out"]), res["pnseg"].cpu().numpy(), res["pterm"].cpu().numpy()))
    (a, sa, ta), (b, sb, tb) = outs
    assert a["counters"] == b["counters"]
    assert np.array_equal(a["exits"], b["exits"])
    assert np.array_equal(sa, sb) and np.array_equal(ta, tb)
    assert np.allclose(a["len"], b["len"], rtol=1e-12, atol=0)
