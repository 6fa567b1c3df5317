"""Seeded, synthetic model specifications for the nested-geometry tracking path.

This module is the ONE input generator shared by the CUDA path (through
``paper_2406_13849_b200.Model.from_spec``) and the CPU oracle (through
``oracle.OracleModel.from_spec``).  It holds no arithmetic of the method: it
only writes down surfaces, materials, cells, universes and arrays as plain
Python data (a JSON-serialisable dict).  Both consumers marshal the dict into
their own builder calls in the same traversal order, so ids agree:

* surfaces, materials: list order;
* universes: list order (CSG, RECT and HEX share one id space);
* cells: global creation order = universes in list order, each CSG universe's
  cells in its own list order.

Geometry follows the paper's model structure (§1 P:133-145 nested
universes; §3 P:193-201 core rect -> assembly rect -> pin; §7.2 P:1318-1363 hex
microreactor) with VERA/BEAVRS-like synthetic dimensions.
Every number below is synthetic input, not a result.
"""
from __future__ import annotations

import copy
import math

KINDS = ("PX", "PY", "PZ", "PLANE", "CZ", "SPHERE")
BCS = ("none", "vacuum", "reflect")

SEED = 240613849          # SURVEY.md §8(d)2 default seed
PARITY_SEEDS = (1, 2, 3)


class Spec:
    """Tiny model-spec builder.  Produces the dict consumed by both sides."""

    def __init__(self, name: str):
        self.name = name
        self.surfaces: list[dict] = []
        self.materials: list[dict] = []
        self.universes: list[dict] = []
        self.root = None
        self.source = None

    # -- primitives --------------------------------------------------------
    def surf(self, kind: str, coef, bc: str = "none") -> int:
        assert kind in KINDS and bc in BCS
        self.surfaces.append({"kind": kind, "coef": [float(c) for c in coef], "bc": bc})
        return len(self.surfaces) - 1

    def mat(self, name: str, sigma_t: float, sigma_a: float, nu_sigma_f: float = 0.0) -> int:
        m = {"name": name, "sigma_t": float(sigma_t), "sigma_a": float(sigma_a)}
        if nu_sigma_f:
            m["nu_sigma_f"] = float(nu_sigma_f)            # one-group fission (reading F1)
        self.materials.append(m)
        return len(self.materials) - 1

    def csg(self, name: str) -> int:
        self.universes.append({"kind": "csg", "name": name, "cells": []})
        return len(self.universes) - 1

    def cell(self, uid: int, hs, material: int | None = None, fill: int | None = None,
             translation=None):
        """hs: list of signed surface references +-(sid+1); + = positive side."""
        u = self.universes[uid]
        assert u["kind"] == "csg"
        assert (material is None) != (fill is None)
        c = {"hs": [int(h) for h in hs]}
        if material is not None:
            c["material"] = int(material)
        else:
            c["fill"] = int(fill)
            if translation is not None:
                c["translation"] = [float(t) for t in translation]
        u["cells"].append(c)

    def rect(self, name: str, ll, pitch, shape, fill, outer: int | None) -> int:
        """Uniform rect array; pitch[2] == 0 -> 2-D (no z index). fill: x fastest."""
        n = shape[0] * shape[1] * shape[2]
        assert len(fill) == n
        self.universes.append({"kind": "rect", "name": name, "ll": [float(v) for v in ll],
                               "pitch": [float(v) for v in pitch], "shape": [int(v) for v in shape],
                               "fill": [int(v) for v in fill],
                               "outer": -1 if outer is None else int(outer)})
        return len(self.universes) - 1

    def rect_edges(self, name: str, edges, fill, outer: int | None) -> int:
        """Non-uniform rect array (Alg. 5 binary-search lattice): edges = [ex, ey, ez]
        strictly increasing mesh divisions per axis; ez = [] -> 2-D.  fill: x fastest."""
        ex, ey, ez = ([float(v) for v in e] for e in edges)
        shape = (len(ex) - 1, len(ey) - 1, max(len(ez) - 1, 1))
        assert len(fill) == shape[0] * shape[1] * shape[2]
        self.universes.append({"kind": "rect", "name": name, "edges": [ex, ey, ez],
                               "shape": list(shape), "fill": [int(v) for v in fill],
                               "outer": -1 if outer is None else int(outer)})
        return len(self.universes) - 1

    def hex(self, name: str, orient: str, center, pitch: float, rings: int, fill,
            outer: int | None, z_lower: float = 0.0, z_pitch: float = 0.0, nz: int = 0) -> int:
        """Hex array (axial q,r).  fill in O9 order: r ascending then q ascending over
        the tiles with max(|q|,|r|,|q+r|) <= rings-1 (times nz layers, z slowest)."""
        assert orient in ("pointy", "flat")
        ntile = 1 + 3 * rings * (rings - 1)
        assert len(fill) == ntile * max(nz, 1)
        self.universes.append({"kind": "hex", "name": name, "orient": orient,
                               "center": [float(center[0]), float(center[1])],
                               "pitch": float(pitch), "rings": int(rings),
                               "z_lower": float(z_lower), "z_pitch": float(z_pitch), "nz": int(nz),
                               "fill": [int(v) for v in fill],
                               "outer": -1 if outer is None else int(outer)})
        return len(self.universes) - 1

    def to_dict(self) -> dict:
        assert self.root is not None and self.source is not None
        return {"name": self.name, "surfaces": copy.deepcopy(self.surfaces),
                "materials": copy.deepcopy(self.materials),
                "universes": copy.deepcopy(self.universes), "root": self.root,
                "source": copy.deepcopy(self.source)}


def hex_tiles(rings: int):
    """(q, r) of the in-lattice tiles in O9 fill order: r ascending, then q ascending."""
    R = rings - 1
    out = []
    for r in range(-R, R + 1):
        for q in range(-R, R + 1):
            if max(abs(q), abs(r), abs(q + r)) <= R:
                out.append((q, r))
    return out


# ---------------------------------------------------------------------------
# shared pieces
# ---------------------------------------------------------------------------
PIN_R = (0.4096, 0.4180, 0.4750)     # fuel / gap / clad outer radii (cm)
GT_R = (0.561, 0.602)                 # guide tube inner / outer radii (cm)
PIN_PITCH = 1.26
ASSY_PITCH = 21.5
ASSY_N = 17
HEIGHT = 365.76

C2_GT = [(2, 5), (2, 8), (2, 11), (3, 3), (3, 13), (5, 2), (5, 5), (5, 8), (5, 11), (5, 14),
         (8, 2), (8, 5), (8, 8), (8, 11), (8, 14), (11, 2), (11, 5), (11, 8), (11, 11), (11, 14),
         (13, 3), (13, 13), (14, 5), (14, 8), (14, 11)]


def _box(sp: Spec, lo, hi, bc):
    """Six axis planes in the canonical order PX-,PX+,PY-,PY+,PZ-,PZ+; returns hs list."""
    ids = [sp.surf("PX", [lo[0]], bc), sp.surf("PX", [hi[0]], bc),
           sp.surf("PY", [lo[1]], bc), sp.surf("PY", [hi[1]], bc),
           sp.surf("PZ", [lo[2]], bc), sp.surf("PZ", [hi[2]], bc)]
    return [ids[0] + 1, -(ids[1] + 1), ids[2] + 1, -(ids[3] + 1), ids[4] + 1, -(ids[5] + 1)]


def _pin(sp: Spec, name, radii, mats):
    """Concentric-CZ pin universe: len(mats) == len(radii)+1 (last = outside)."""
    u = sp.csg(name)
    cz = [sp.surf("CZ", [0.0, 0.0, r]) for r in radii]
    for i, m in enumerate(mats):
        hs = []
        if i > 0:
            hs.append(cz[i - 1] + 1)
        if i < len(radii):
            hs.append(-(cz[i] + 1))
        sp.cell(u, hs, material=m)
    return u


def _pwr_materials(sp: Spec, uniform=None):
    def m(name, st, sa):
        if uniform is not None:
            st, sa = uniform
        return sp.mat(name, st, sa)
    return {"uo2": m("uo2", 0.60, 0.12), "gap": m("gap", 0.0, 0.0), "zr": m("zr", 0.30, 0.003),
            "water": m("water", 1.20, 0.02)}


# ---------------------------------------------------------------------------
# C1: pincell (configs[0])
# ---------------------------------------------------------------------------
def c1_pincell(bc="reflect", uniform=None, void=False) -> dict:
    """Single UO2 pin (fuel/gap/clad cylinders) in a reflective water square.
    uniform=(st, sa): every material set to the same (P9 volume recovery).
    void=True: every material void (P8 chord invariant)."""
    name = "c1_pincell" + ("_void" if void else "") + ("_uniform" if uniform else "")
    sp = Spec(name)
    if void:
        uniform = (0.0, 0.0)
    hp = PIN_PITCH / 2
    root = sp.csg("root")
    box = _box(sp, (-hp, -hp, 0.0), (hp, hp, HEIGHT), bc)
    mats = _pwr_materials(sp, uniform)
    pin = _pin(sp, "pin", PIN_R, [mats["uo2"], mats["gap"], mats["zr"], mats["water"]])
    sp.cell(root, box, fill=pin)
    sp.root = root
    sp.source = {"lo": [-hp, -hp, 0.0], "hi": [hp, hp, HEIGHT]}
    return sp.to_dict()


def with_fission(spec: dict, nu_sigma_f: dict) -> dict:
    """Copy of a model spec with one-group nu Sigma_f on the named materials (reading F1)."""
    out = copy.deepcopy(spec)
    for m in out["materials"]:
        if m["name"] in nu_sigma_f:
            m["nu_sigma_f"] = float(nu_sigma_f[m["name"]])
    return out


# ---------------------------------------------------------------------------
# C2: 17x17 assembly (configs[1])
# ---------------------------------------------------------------------------
def _assembly(sp: Spec, name, fuel_pin, gt_pin, water_pin, gt_pos=C2_GT):
    fill = []
    gts = set(gt_pos)
    for j in range(ASSY_N):          # row (y)
        for i in range(ASSY_N):      # col (x), x fastest
            fill.append(gt_pin if (j, i) in gts else fuel_pin)
    ll = -ASSY_N * PIN_PITCH / 2
    return sp.rect(name, (ll, ll, 0.0), (PIN_PITCH, PIN_PITCH, 0.0), (ASSY_N, ASSY_N, 1), fill,
                   water_pin)


def c2_assembly() -> dict:
    sp = Spec("c2_assembly")
    root = sp.csg("root")
    ha = ASSY_PITCH / 2
    box = _box(sp, (-ha, -ha, 0.0), (ha, ha, HEIGHT), "reflect")
    mats = _pwr_materials(sp)
    fuel = _pin(sp, "fuel_pin", PIN_R, [mats["uo2"], mats["gap"], mats["zr"], mats["water"]])
    gt = _pin(sp, "guide_tube", GT_R, [mats["water"], mats["zr"], mats["water"]])
    water = _pin(sp, "water_pin", (), [mats["water"]])
    assy = _assembly(sp, "assembly", fuel, gt, water)
    sp.cell(root, box, fill=assy)
    sp.root = root
    sp.source = {"lo": [-ha, -ha, 0.0], "hi": [ha, ha, HEIGHT]}
    return sp.to_dict()


def c2_gap_assembly() -> dict:
    """C2 as a NON-UNIFORM 19x19 lattice (the paper's motivation for Alg. 5's binary search,
    P:500-505): a 0.04 cm water-gap column / row on each side of the 17 pin pitches, filled by
    the water pin, instead of the uniform lattice's `outer`.  The material layout is exactly
    C2's, and the 17x17 edges are computed like the uniform edges (ll + i*p)."""
    sp = Spec("c2_gap_assembly")
    root = sp.csg("root")
    ha = ASSY_PITCH / 2
    box = _box(sp, (-ha, -ha, 0.0), (ha, ha, HEIGHT), "reflect")
    mats = _pwr_materials(sp)
    fuel = _pin(sp, "fuel_pin", PIN_R, [mats["uo2"], mats["gap"], mats["zr"], mats["water"]])
    gt = _pin(sp, "guide_tube", GT_R, [mats["water"], mats["zr"], mats["water"]])
    water = _pin(sp, "water_pin", (), [mats["water"]])
    ll = -ASSY_N * PIN_PITCH / 2
    e = [-ha] + [ll + i * PIN_PITCH for i in range(ASSY_N + 1)] + [ha]
    gts = set(C2_GT)
    fill = []
    for j in range(ASSY_N + 2):
        for i in range(ASSY_N + 2):
            inner = 1 <= i <= ASSY_N and 1 <= j <= ASSY_N
            fill.append((gt if (j - 1, i - 1) in gts else fuel) if inner else water)
    assy = sp.rect_edges("gap_assembly", [e, e, []], fill, water)
    sp.cell(root, box, fill=assy)
    sp.root = root
    sp.source = {"lo": [-ha, -ha, 0.0], "hi": [ha, ha, HEIGHT]}
    return sp.to_dict()


def gap_lattice(nonuniform: bool) -> dict:
    """5x5 pin lattice, pitch 1.25, with a 0.0625 cm water gap to a reflective box: either a
    uniform lattice whose `outer` (water pin) fills the gap, or a NON-UNIFORM 7x7 lattice with
    explicit gap columns.  All divisions and tile centres are dyadic, hence exact in both forms,
    so the two walks must be bit-identical (pin for reading N1)."""
    sp = Spec("gap_lattice_" + ("nonuniform" if nonuniform else "uniform"))
    root = sp.csg("root")
    n, p, g = 5, 1.25, 0.0625
    ll = -n * p / 2
    h = -ll + g
    box = _box(sp, (-h, -h, 0.0), (h, h, 10.0), "reflect")
    mats = _pwr_materials(sp)
    fuel = _pin(sp, "fuel_pin", PIN_R, [mats["uo2"], mats["gap"], mats["zr"], mats["water"]])
    gt = _pin(sp, "guide_tube", GT_R, [mats["water"], mats["zr"], mats["water"]])
    water = _pin(sp, "water_pin", (), [mats["water"]])
    pin = lambda i, j: gt if (i + j) % 3 == 0 else fuel          # noqa: E731
    if nonuniform:
        e = [-h] + [ll + i * p for i in range(n + 1)] + [h]
        fill = [pin(i - 1, j - 1) if 1 <= i <= n and 1 <= j <= n else water
                for j in range(n + 2) for i in range(n + 2)]
        lat = sp.rect_edges("lattice", [e, e, []], fill, water)
    else:
        lat = sp.rect("lattice", (ll, ll, 0.0), (p, p, 0.0), (n, n, 1),
                      [pin(i, j) for j in range(n) for i in range(n)], water)
    sp.cell(root, box, fill=lat)
    sp.root = root
    sp.source = {"lo": [-h, -h, 0.0], "hi": [h, h, 10.0]}
    return sp.to_dict()


def nonuniform_slabs(sigma_t=1.0, sigma_a=0.1) -> dict:
    """Reflective box [0,6]x[0,3]x[0,2] tiled by a non-uniform 3x2x2 lattice (x edges 0,1,3,6;
    y 0,0.5,3; z 0,0.7,2), one all-space cell of the same material per tile: track-length
    fractions must equal the tile volumes (P9 applied to Alg. 5 lattices)."""
    sp = Spec("nonuniform_slabs")
    root = sp.csg("root")
    box = _box(sp, (0.0, 0.0, 0.0), (6.0, 3.0, 2.0), "reflect")
    m = sp.mat("medium", sigma_t, sigma_a)
    tiles = []
    for t in range(12):
        u = sp.csg(f"tile{t}")
        sp.cell(u, [], material=m)
        tiles.append(u)
    lat = sp.rect_edges("slabs", [[0.0, 1.0, 3.0, 6.0], [0.0, 0.5, 3.0], [0.0, 0.7, 2.0]], tiles, None)
    sp.cell(root, box, fill=lat)
    sp.root = root
    sp.source = {"lo": [0.0, 0.0, 0.0], "hi": [6.0, 3.0, 2.0]}
    return sp.to_dict()


# ---------------------------------------------------------------------------
# C3: full-core PWR (the metric's config)
# ---------------------------------------------------------------------------
C3_ROW_WIDTHS = (7, 11, 13, 13, 15, 15, 15, 15, 15, 15, 15, 13, 13, 11, 7)
C3_RADII = (185.0, 187.5, 187.96, 193.68, 219.15, 240.8)   # baffle .. vessel outer


def c3_loading():
    """15x15 core map: 0 = empty (water assembly), 1..3 = enrichment type.
    Row widths 7,11,13,13,15x7,13,13,11,7 -> 193 assemblies."""
    n = 15
    grid = [[0] * n for _ in range(n)]
    for j, w in enumerate(C3_ROW_WIDTHS):
        i0 = (n - w) // 2
        for i in range(i0, i0 + w):
            grid[j][i] = 1
    # periphery (a loaded position with an empty 4-neighbour) -> type 3;
    # interior checkerboard of types 1 / 2
    for j in range(n):
        for i in range(n):
            if grid[j][i] == 0:
                continue
            edge = any(not (0 <= j + dj < n and 0 <= i + di < n) or grid[j + dj][i + di] == 0
                       for dj, di in ((1, 0), (-1, 0), (0, 1), (0, -1)))
            grid[j][i] = 3 if edge else (1 if (i + j) % 2 == 0 else 2)
    return grid


def c3_full_core() -> dict:
    sp = Spec("c3_full_core")
    root = sp.csg("root")
    # canonical root surface order: PZ-, PZ+, then CZs ascending (rect-tracker gate)
    pz0 = sp.surf("PZ", [0.0], "vacuum")
    pz1 = sp.surf("PZ", [HEIGHT], "vacuum")
    cz = [sp.surf("CZ", [0.0, 0.0, r], "vacuum" if r == C3_RADII[-1] else "none")
          for r in C3_RADII]
    fuel_m = [sp.mat("uo2_a", 0.60, 0.10), sp.mat("uo2_b", 0.60, 0.12), sp.mat("uo2_c", 0.60, 0.14)]
    gap = sp.mat("gap", 0.0, 0.0)
    zr = sp.mat("zr", 0.30, 0.003)
    water = sp.mat("water", 1.20, 0.02)
    steel = sp.mat("steel", 0.90, 0.05)

    fuel_pins = [_pin(sp, f"fuel_pin_{e}", PIN_R, [fuel_m[e], gap, zr, water]) for e in range(3)]
    gt = _pin(sp, "guide_tube", GT_R, [water, zr, water])
    water_pin = _pin(sp, "water_pin", (), [water])
    assys = [_assembly(sp, f"assembly_{e}", fuel_pins[e], gt, water_pin) for e in range(3)]
    ll = -ASSY_N * PIN_PITCH / 2
    water_assy = sp.rect("water_assembly", (ll, ll, 0.0), (PIN_PITCH, PIN_PITCH, 0.0),
                         (ASSY_N, ASSY_N, 1), [water_pin] * (ASSY_N * ASSY_N), water_pin)
    grid = c3_loading()
    fill = []
    for j in range(15):
        for i in range(15):
            t = grid[j][i]
            fill.append(water_assy if t == 0 else assys[t - 1])
    core_ll = -15 * ASSY_PITCH / 2
    core = sp.rect("core", (core_ll, core_ll, 0.0), (ASSY_PITCH, ASSY_PITCH, 0.0), (15, 15, 1),
                   fill, water_assy)
    zs = [pz0 + 1, -(pz1 + 1)]
    sp.cell(root, [-(cz[0] + 1)] + zs, fill=core)
    ring_mats = [steel, water, steel, water, steel]   # baffle, water, barrel, downcomer, vessel
    for k, m in enumerate(ring_mats):
        sp.cell(root, [cz[k] + 1, -(cz[k + 1] + 1)] + zs, material=m)
    sp.root = root
    sp.source = {"lo": [core_ll, core_ll, 0.0], "hi": [-core_ll, -core_ll, HEIGHT]}
    return sp.to_dict()


# ---------------------------------------------------------------------------
# C4: hexagonal microreactor (generic tracker only)
# ---------------------------------------------------------------------------
C4_HEIGHT = 150.0


def c4_hex_microreactor() -> dict:
    sp = Spec("c4_hex_microreactor")
    root = sp.csg("root")
    pz0 = sp.surf("PZ", [0.0], "vacuum")
    pz1 = sp.surf("PZ", [C4_HEIGHT], "vacuum")
    cz_core = sp.surf("CZ", [0.0, 0.0, 80.0])
    cz_out = sp.surf("CZ", [0.0, 0.0, 110.0], "vacuum")
    un = sp.mat("UN", 0.55, 0.15)
    yh = sp.mat("YH", 1.6, 0.01)
    hp = sp.mat("heat_pipe", 0.3, 0.02)
    matrix = sp.mat("matrix", 0.9, 0.05)
    beo = sp.mat("BeO", 0.9, 0.002)
    absorber = sp.mat("absorber", 2.0, 1.8)
    void = sp.mat("void", 0.0, 0.0)
    clad = sp.mat("clad", 0.7, 0.01)

    fuel_pin = _pin(sp, "fuel_pin", (0.70, 0.75), [un, clad, matrix])
    mod_pin = _pin(sp, "moderator_pin", (0.80, 0.85), [yh, clad, matrix])
    hp_pin = _pin(sp, "heat_pipe", (0.80,), [hp, matrix])
    matrix_u = _pin(sp, "matrix", (), [matrix])
    void_u = _pin(sp, "void", (), [void])
    refl_u = _pin(sp, "reflector", (), [beo])
    cls = {0: hp_pin, 1: fuel_pin, 2: mod_pin}
    afill = [cls[(q - r) % 3] for (q, r) in hex_tiles(9)]
    assy = sp.hex("assembly", "pointy", (0.0, 0.0), 1.9, 9, afill, matrix_u)
    cfill = [void_u if (q, r) == (0, 0) else assy for (q, r) in hex_tiles(3)]
    core = sp.hex("core", "flat", (0.0, 0.0), 30.0, 3, cfill, refl_u)

    zs = [pz0 + 1, -(pz1 + 1)]
    sp.cell(root, [-(cz_core + 1)] + zs, fill=core)
    refl_hs = [cz_core + 1, -(cz_out + 1)] + zs
    for k in range(12):
        a = math.radians(15.0 + 30.0 * k)
        cx, cy = 95.0 * math.cos(a), 95.0 * math.sin(a)
        c9 = sp.surf("CZ", [cx, cy, 9.0])
        c10 = sp.surf("CZ", [cx, cy, 10.0])
        pl = sp.surf("PLANE", [math.cos(a), math.sin(a), 0.0, 95.0])
        sp.cell(root, [-(c9 + 1)] + zs, material=beo)
        sp.cell(root, [c9 + 1, -(c10 + 1), -(pl + 1)] + zs, material=absorber)
        sp.cell(root, [c9 + 1, -(c10 + 1), pl + 1] + zs, material=beo)
        refl_hs.append(c10 + 1)
    sp.cell(root, refl_hs, material=beo)
    sp.root = root
    sp.source = {"lo": [-75.0, -75.0, 0.0], "hi": [75.0, 75.0, C4_HEIGHT]}
    return sp.to_dict()


# ---------------------------------------------------------------------------
# C5: deep nesting, mixed (C5m) and rect-only (C5r)
# ---------------------------------------------------------------------------
def c5_deep(mixed: bool) -> dict:
    sp = Spec("c5m_deep_mixed" if mixed else "c5r_deep_rect")
    root = sp.csg("root")
    box = _box(sp, (-45.0, -45.0, 0.0), (45.0, 45.0, 100.0), "reflect")
    mats = _pwr_materials(sp)
    fuel = _pin(sp, "fuel_pin", PIN_R, [mats["uo2"], mats["gap"], mats["zr"], mats["water"]])
    gt = _pin(sp, "guide_tube", GT_R, [mats["water"], mats["zr"], mats["water"]])
    water_pin = _pin(sp, "water_pin", (), [mats["water"]])
    p5 = [gt if (i, j) == (2, 2) else fuel for j in range(5) for i in range(5)]
    l5 = -5 * PIN_PITCH / 2
    r5 = sp.rect("rect5x5", (l5, l5, 0.0), (PIN_PITCH, PIN_PITCH, 0.0), (5, 5, 1), p5, water_pin)
    if mixed:
        mid = sp.hex("hex7", "flat", (0.0, 0.0), 9.0, 2, [r5] * 7, water_pin)
    else:
        water5 = sp.rect("water5x5", (l5, l5, 0.0), (PIN_PITCH, PIN_PITCH, 0.0), (5, 5, 1),
                         [water_pin] * 25, water_pin)
        mid = sp.rect("rect3x3_mid", (-13.5, -13.5, 0.0), (9.0, 9.0, 0.0), (3, 3, 1), [r5] * 9,
                      water5)
    top = sp.rect("rect3x3_top", (-45.0, -45.0, 0.0), (30.0, 30.0, 0.0), (3, 3, 1), [mid] * 9, None)
    sp.cell(root, box, fill=top)
    sp.root = root
    sp.source = {"lo": [-45.0, -45.0, 0.0], "hi": [45.0, 45.0, 100.0]}
    return sp.to_dict()


# ---------------------------------------------------------------------------
# test models (P8-P12, O13)
# ---------------------------------------------------------------------------
def infinite_medium(sigma_t=1.0, sigma_a=0.25, nu_sigma_f=0.0) -> dict:
    """One material in an all-REFLECT box (P10): track length per history ~ Exp(Sigma_a).
    With nu_sigma_f: k_inf = nu Sigma_f / Sigma_a (F1)."""
    sp = Spec("infinite_medium")
    root = sp.csg("root")
    box = _box(sp, (-1.0, -1.0, -1.0), (1.0, 1.0, 1.0), "reflect")
    m = sp.mat("m", sigma_t, sigma_a, nu_sigma_f)
    sp.cell(root, box, material=m)
    sp.root = root
    sp.source = {"lo": [-1.0, -1.0, -1.0], "hi": [1.0, 1.0, 1.0]}
    return sp.to_dict()


def lattice3_nested(flat=False) -> dict:
    """3x3 pin lattice: nested (root -> RECT -> pin) or the same geometry as ONE flat
    CSG universe (planes at LL+i*p, cylinders at tile centres) -- P12.  The pitch 1.25
    is a binary fraction so the lattice edge LL+3p coincides exactly with the box wall."""
    sp = Spec("lattice3_flat" if flat else "lattice3_nested")
    root = sp.csg("root")
    p = 1.25
    ll = -1.5 * p
    box = _box(sp, (ll, ll, 0.0), (-ll, -ll, 10.0), "reflect")
    mats = _pwr_materials(sp)
    pm = [mats["uo2"], mats["gap"], mats["zr"], mats["water"]]
    if not flat:
        pin = _pin(sp, "pin", PIN_R, pm)
        lat = sp.rect("lat", (ll, ll, 0.0), (p, p, 0.0), (3, 3, 1), [pin] * 9, None)
        sp.cell(root, box, fill=lat)
    else:
        # planes at the lattice edges (interior only; the box supplies the outer ones)
        px = [sp.surf("PX", [ll + i * p]) for i in (1, 2)]
        py = [sp.surf("PY", [ll + j * p]) for j in (1, 2)]
        xb = [box[0], None, None, box[1]]
        yb = [box[2], None, None, box[3]]
        for j in range(3):
            for i in range(3):
                cx = ll + (i + 0.5) * p
                cy = ll + (j + 0.5) * p
                czs = [sp.surf("CZ", [cx, cy, r]) for r in PIN_R]
                walls = [box[4], box[5]]
                walls.append(xb[0] if i == 0 else px[i - 1] + 1)
                walls.append(xb[3] if i == 2 else -(px[i] + 1))
                walls.append(yb[0] if j == 0 else py[j - 1] + 1)
                walls.append(yb[3] if j == 2 else -(py[j] + 1))
                for k, m in enumerate(pm):
                    hs = list(walls)
                    if k > 0:
                        hs.append(czs[k - 1] + 1)
                    if k < 3:
                        hs.append(-(czs[k] + 1))
                    sp.cell(root, hs, material=m)
    sp.root = root
    sp.source = {"lo": [ll, ll, 0.0], "hi": [-ll, -ll, 10.0]}
    return sp.to_dict()


def sphere_in_box() -> dict:
    """A sphere and a tilted PLANE inside a vacuum box: exercises SPHERE/PLANE code."""
    sp = Spec("sphere_in_box")
    root = sp.csg("root")
    box = _box(sp, (-2.0, -2.0, -2.0), (2.0, 2.0, 2.0), "vacuum")
    s = sp.surf("SPHERE", [0.1, -0.2, 0.05, 1.3])
    pl = sp.surf("PLANE", [0.3, 0.4, 0.5, 0.2])
    a = sp.mat("a", 0.8, 0.2)
    b = sp.mat("b", 0.4, 0.1)
    c = sp.mat("c", 1.1, 0.5)
    sp.cell(root, box + [-(s + 1), -(pl + 1)], material=a)
    sp.cell(root, box + [-(s + 1), pl + 1], material=b)
    sp.cell(root, box + [s + 1], material=c)
    sp.root = root
    sp.source = {"lo": [-2.0, -2.0, -2.0], "hi": [2.0, 2.0, 2.0]}
    return sp.to_dict()


def slab_mix() -> dict:
    """Axis-plane pairings for the slab-pair evaluation (DESIGN §5 "Slab pairs"): adjacent
    opposite-sense pairs of one axis (slabs), a same-axis pair that is not adjacent in the canonical
    order, same-sense planes, four PX planes in one cell, a cylinder, reflective PX walls."""
    sp = Spec("slab_mix")
    root = sp.csg("root")
    px0, px1 = sp.surf("PX", [-3.0], "reflect"), sp.surf("PX", [3.0], "reflect")
    py0, py1 = sp.surf("PY", [-3.0], "vacuum"), sp.surf("PY", [3.0], "vacuum")
    pz0, pz1 = sp.surf("PZ", [-3.0], "vacuum"), sp.surf("PZ", [3.0], "vacuum")
    box = [px0 + 1, -(px1 + 1), py0 + 1, -(py1 + 1), pz0 + 1, -(pz1 + 1)]
    x0 = sp.surf("PX", [0.0])
    xm1 = sp.surf("PX", [-1.0])
    y1 = sp.surf("PY", [1.0])
    x15 = sp.surf("PX", [1.5])
    cz = sp.surf("CZ", [2.0, 2.0, 0.5])
    m = [sp.mat(f"m{k}", 0.3 + 0.25 * k, 0.05 + 0.02 * k) for k in range(6)]
    sp.cell(root, box + [-(x0 + 1), xm1 + 1], material=m[0])                  # -1 <= x < 0: two PX slabs
    sp.cell(root, box + [-(xm1 + 1)], material=m[1])                          # x < -1
    sp.cell(root, box + [x0 + 1, -(y1 + 1), -(x15 + 1)], material=m[2])       # PX pair not adjacent
    sp.cell(root, box + [x0 + 1, -(y1 + 1), x15 + 1], material=m[3])          # same-sense PX planes
    sp.cell(root, box + [x0 + 1, y1 + 1, cz + 1], material=m[4])
    sp.cell(root, box + [x0 + 1, y1 + 1, -(cz + 1)], material=m[5])
    sp.root = root
    sp.source = {"lo": [-3.0, -3.0, -3.0], "hi": [3.0, 3.0, 3.0]}
    return sp.to_dict()


def hex_pins_small(orient="pointy") -> dict:
    """Small 3-ring hex lattice of pins in a reflective box with a 3-D z stack."""
    sp = Spec("hex_small_" + orient)
    root = sp.csg("root")
    box = _box(sp, (-4.0, -4.0, 0.0), (4.0, 4.0, 6.0), "reflect")
    mats = _pwr_materials(sp)
    fuel = _pin(sp, "fuel_pin", (0.5, 0.55), [mats["uo2"], mats["zr"], mats["water"]])
    gt = _pin(sp, "gt", (0.5,), [mats["water"], mats["zr"]])
    water = _pin(sp, "water", (), [mats["water"]])
    tiles = hex_tiles(3)
    fill = []
    for kz in range(2):
        for (q, r) in tiles:
            fill.append(gt if (q - r + kz) % 3 == 0 else fuel)
    lat = sp.hex("lat", orient, (0.1, -0.05), 1.6, 3, fill, water, z_lower=0.5, z_pitch=2.5, nz=2)
    sp.cell(root, box, fill=lat)
    sp.root = root
    sp.source = {"lo": [-4.0, -4.0, 0.0], "hi": [4.0, 4.0, 6.0]}
    return sp.to_dict()


def rect3d_small() -> dict:
    """A 3-D rect lattice (z-indexed) with translated CSG fills: exercises RECT z walls,
    translations and a non-centred lattice."""
    sp = Spec("rect3d_small")
    root = sp.csg("root")
    box = _box(sp, (-3.0, -2.0, -1.0), (3.5, 2.5, 4.0), "vacuum")
    mats = _pwr_materials(sp)
    pin = _pin(sp, "pin", (0.3, 0.45), [mats["uo2"], mats["zr"], mats["water"]])
    blk = sp.csg("block")
    s = sp.surf("SPHERE", [0.0, 0.0, 0.0, 0.4])
    sp.cell(blk, [-(s + 1)], material=mats["zr"])
    sp.cell(blk, [s + 1], material=mats["water"])
    fill = [pin if (i + j + k) % 2 == 0 else blk for k in range(3) for j in range(3) for i in range(4)]
    lat = sp.rect("lat3d", (-2.6, -1.7, -0.8), (1.3, 1.25, 1.5), (4, 3, 3), fill, blk)
    sp.cell(root, box, fill=lat, translation=(0.2, 0.1, 0.0))
    sp.root = root
    sp.source = {"lo": [-3.0, -2.0, -1.0], "hi": [3.5, 2.5, 4.0]}
    return sp.to_dict()


# ---------------------------------------------------------------------------
# O13 / O16 test models: near-coincident surfaces (PAPER.md:554-556 removes coincident lower-level
# surfaces in preprocessing; this build keeps them and flags histories that come within 1e-10 cm)
# ---------------------------------------------------------------------------
NEAR_GAP = 5e-11           # cm: second surface this far inside the first (O16 flags fire at <= 1e-10)
NEAR_BODY = 0.3            # body radius / plane offset (cm); 2R != 1 so the 2R scale of the tolerance shows
NEAR_PLANE_N = (1.0, 2.0, 2.0)   # |n| = 3: exercises the 1e-10 |n| tolerance of an unnormalised PLANE


def near_coincident(kind: str = "CZ", gap: float = NEAR_GAP, void: bool = False,
                    body=(0.5, 0.05), outside=(0.3, 0.03)) -> dict:
    """A body bounded by surface S inside a vacuum box [-1, 1]^3; the outside cell also carries a
    second surface S' lying `gap` cm inside S (a redundant half-space: outside S implies outside
    S').  Leaving the body through S lands `gap` from S' (O16 F1 on the new cell); entering it
    meets S and then S' about `gap` further on (F2).  kind: CZ (R = 0.3 about the z axis), SPHERE
    (R = 0.3 about the origin) or PLANE (n = (1, 2, 2), n.r = 0.9: the body is n.r < 0.9).
    void=True: both materials void (deterministic rays)."""
    sp = Spec(f"near_{kind.lower()}" + ("_void" if void else "") + ("" if gap == NEAR_GAP else f"_{gap:g}"))
    root = sp.csg("root")
    box = _box(sp, (-1.0, -1.0, -1.0), (1.0, 1.0, 1.0), "vacuum")
    R = NEAR_BODY
    if kind == "CZ":
        s0 = sp.surf("CZ", [0.0, 0.0, R])
        s1 = sp.surf("CZ", [0.0, 0.0, R - gap])
    elif kind == "SPHERE":
        s0 = sp.surf("SPHERE", [0.0, 0.0, 0.0, R])
        s1 = sp.surf("SPHERE", [0.0, 0.0, 0.0, R - gap])
    else:
        nn = NEAR_PLANE_N
        norm = math.sqrt(sum(v * v for v in nn))
        s0 = sp.surf("PLANE", [nn[0], nn[1], nn[2], norm * R])
        s1 = sp.surf("PLANE", [nn[0], nn[1], nn[2], norm * (R - gap)])
    if void:
        body, outside = (0.0, 0.0), (0.0, 0.0)
    mb = sp.mat("body", *body)
    mo = sp.mat("outside", *outside)
    sp.cell(root, box + [-(s0 + 1)], material=mb)
    sp.cell(root, box + [s0 + 1, s1 + 1], material=mo)
    sp.root = root
    sp.source = {"lo": [-1.0, -1.0, -1.0], "hi": [1.0, 1.0, 1.0]}
    return sp.to_dict()


def grazing_lattice(gap: float = NEAR_GAP, void: bool = False) -> dict:
    """3x3 pin lattice (pitch 1.25, reflective box on the lattice edges) whose pin universe splits
    the moderator with a PX plane `gap` cm inside the tile's +x wall: a CSG surface grazing a lattice
    wall one level up.  Moving +x in the moderator, the plane and the wall are `gap`/u apart (F2
    across levels); entering a tile through its +x wall descends `gap` from the plane (F1)."""
    sp = Spec("grazing_lattice" + ("_void" if void else "") + ("" if gap == NEAR_GAP else f"_{gap:g}"))
    root = sp.csg("root")
    p = 1.25
    ll = -1.5 * p
    box = _box(sp, (ll, ll, 0.0), (-ll, -ll, 10.0), "reflect")
    mats = _pwr_materials(sp, uniform=(0.0, 0.0) if void else None)
    pin = sp.csg("pin")
    cz = [sp.surf("CZ", [0.0, 0.0, r]) for r in (0.4096, 0.475)]
    px = sp.surf("PX", [0.5 * p - gap])
    sp.cell(pin, [-(cz[0] + 1)], material=mats["uo2"])
    sp.cell(pin, [cz[0] + 1, -(cz[1] + 1)], material=mats["zr"])
    sp.cell(pin, [cz[1] + 1, -(px + 1)], material=mats["water"])
    sp.cell(pin, [cz[1] + 1, px + 1], material=mats["water"])
    lat = sp.rect("lat", (ll, ll, 0.0), (p, p, 0.0), (3, 3, 1), [pin] * 9, None)
    sp.cell(root, box, fill=lat)
    sp.root = root
    sp.source = {"lo": [ll, ll, 0.0], "hi": [-ll, -ll, 10.0]}
    return sp.to_dict()


CONFIGS = {
    "c1": (c1_pincell, 10_000),
    "c2": (c2_assembly, 10_000_000),
    "c3": (c3_full_core, 100_000_000),
    "c4": (c4_hex_microreactor, 100_000_000),
    "c5m": (lambda: c5_deep(True), 10_000_000),
    "c5r": (lambda: c5_deep(False), 10_000_000),
}


def config(name: str) -> tuple[dict, int]:
    """(model spec, BASELINE.json particle count) for a config name."""
    fn, n = CONFIGS[name]
    return fn(), n
