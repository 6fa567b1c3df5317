"""CPU oracle for the nested-geometry tracking path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package.  It loads ``liboracle.so``
(plain C, ``oracle/oracle.c``, -O2 -ffp-contract=off -fopenmp) and marshals the
``workloads`` model spec into it.  It shares no code with
``paper_2406_13849_b200`` (the CUDA path) and neither imports the other.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "oracle.c")
LIB = os.path.join(HERE, "liboracle.so")

KIND = {"PX": 0, "PY": 1, "PZ": 2, "PLANE": 3, "CZ": 4, "SPHERE": 5}
BC = {"none": 0, "vacuum": 1, "reflect": 2}
COUNTERS = ["particles", "segments", "crossings", "reflections", "leaks", "collisions",
            "absorptions", "lost", "capped", "flagged"] + [f"cross_l{i}" for i in range(8)]
NC = len(COUNTERS)
EVAL_KINDS = ["axis", "plane", "cz", "sphere", "rect", "hex"]
# LINPACK-weighted fp64 flops per distance candidate
EVAL_FLOPS = {"axis": 2, "plane": 12, "cz": 18, "sphere": 19, "rect": 2, "hex": 32}

TRACE_DTYPE = np.dtype([("pid", "<u8"), ("s", "<f8"), ("seg", "<u4"), ("cell_before", "<i4"),
                        ("cell_after", "<i4"), ("j", "<i4"), ("kind", "u1"), ("level", "i1"),
                        ("terminal", "u1"), ("pad", "u1"), ("flags", "<u4")])


def build(force: bool = False) -> str:
    """Compile liboracle.so (building the checker is not using it)."""
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        cmd = ["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fopenmp",
               "-fPIC", "-shared", "-Wall", "-o", LIB + ".tmp", SRC, "-lm"]
        subprocess.check_call(cmd)
        os.replace(LIB + ".tmp", LIB)
    return LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(LIB)
        vp, i32, u64, dp = C.c_void_p, C.c_int, C.c_uint64, C.c_void_p
        L.orc_model_new.restype = vp
        L.orc_model_free.argtypes = [vp]
        L.orc_add_surface.argtypes = [vp, i32, dp, i32]
        L.orc_add_material.argtypes = [vp, C.c_double, C.c_double]
        L.orc_add_csg_universe.argtypes = [vp]
        L.orc_add_cell.argtypes = [vp, i32, dp, i32, i32, i32, dp]
        L.orc_add_rect.argtypes = [vp, dp, dp, dp, dp, i32]
        L.orc_add_rect_edges.argtypes = [vp, dp, dp, dp, i32]
        L.orc_add_hex.argtypes = [vp, i32, dp, C.c_double, i32, C.c_double, C.c_double, i32, dp, i32]
        L.orc_set_root.argtypes = [vp, i32]
        L.orc_finalize.argtypes = [vp]
        for f in ("orc_n_material_cells", "orc_out_len", "orc_max_depth"):
            getattr(L, f).argtypes = [vp]
        L.orc_material_cell_ids.argtypes = [vp, dp]
        L.orc_cell_material.argtypes = [vp, i32]
        L.orc_run.argtypes = [vp, u64, u64, u64, dp, dp, u64, i32, dp, dp, dp, u64, dp, dp, dp, dp, dp, dp, dp, dp]
        L.orc_run_states.argtypes = [vp, u64, u64, u64, dp, u64, i32, dp, dp, dp, u64, dp, dp, dp, dp, dp, dp, dp, dp]
        L.orc_set_fission.argtypes = [vp, i32, C.c_double]
        L.orc_max_sites.argtypes = [vp]
        L.orc_fission_source.argtypes = [vp, dp, dp, u64, u64, C.c_uint32, u64, dp]
        L.orc_fission_source.restype = u64
        L.orc_source_from_sites.argtypes = [dp, u64, u64, C.c_uint32, u64, u64, dp]
        L.orc_n_instances.argtypes = [vp]
        L.orc_n_instances.restype = C.c_long
        L.orc_instance_cells.argtypes = [vp, dp]
        L.orc_instance_cells.restype = C.c_long
        L.orc_set_mesh.argtypes = [vp, dp, dp, dp]
        L.orc_find_cells.argtypes = [vp, dp, u64, dp, dp]
        L.orc_count_containing.argtypes = [vp, i32, dp]
        L.orc_surface_distance.argtypes = [vp, i32, i32, i32, dp, dp]
        L.orc_surface_distance.restype = C.c_double
        L.orc_surface_f.argtypes = [vp, i32, dp]
        L.orc_surface_f.restype = C.c_double
        L.orc_locate_array.argtypes = [vp, i32, dp, dp, dp, dp, dp]
        L.orc_hex_owns.argtypes = [vp, i32, i32, i32, dp]
        L.orc_philox.argtypes = [dp, dp, dp]
        L.orc_u01.argtypes = [C.c_uint32, C.c_uint32]
        L.orc_u01.restype = C.c_double
        L.orc_log.argtypes = [C.c_double]
        L.orc_log.restype = C.c_double
        L.orc_sincos2pi.argtypes = [C.c_double, dp, dp]
        assert L.orc_trace_rec_size() == TRACE_DTYPE.itemsize
        assert L.orc_ncount() == NC
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def philox(ctr, key):
    c = np.asarray(ctr, dtype=np.uint32)
    k = np.asarray(key, dtype=np.uint32)
    o = np.zeros(4, dtype=np.uint32)
    lib().orc_philox(_p(c), _p(k), _p(o))
    return o


def u01(h: int, l: int) -> float:
    return lib().orc_u01(h, l)


def log(x: float) -> float:
    return lib().orc_log(x)


def iso(xmu: float, xphi: float) -> np.ndarray:
    """O15 isotropic direction of one (xi_mu, xi_phi) draw pair."""
    L = lib()
    L.orc_iso.argtypes = [C.c_double, C.c_double, C.c_void_p]
    om = np.zeros(3)
    L.orc_iso(xmu, xphi, _p(om))
    return om


def sincos2pi(xi: float):
    c = np.zeros(1)
    s = np.zeros(1)
    lib().orc_sincos2pi(xi, _p(c), _p(s))
    return float(c[0]), float(s[0])


class OracleModel:
    """Oracle model built from a workloads spec (same traversal order as the product)."""

    def __init__(self):
        self.L = lib()
        self.h = self.L.orc_model_new()
        self.spec = None

    def __del__(self):
        try:
            self.L.orc_model_free(self.h)
        except Exception:
            pass

    @classmethod
    def from_spec(cls, spec: dict) -> "OracleModel":
        m = cls()
        L = m.L
        m.spec = spec
        for s in spec["surfaces"]:
            coef = np.zeros(4)
            coef[:len(s["coef"])] = s["coef"]
            r = L.orc_add_surface(m.h, KIND[s["kind"]], _p(coef), BC[s["bc"]])
            assert r >= 0
        for mt in spec["materials"]:
            k = L.orc_add_material(m.h, mt["sigma_t"], mt["sigma_a"])
            if mt.get("nu_sigma_f", 0.0):
                if L.orc_set_fission(m.h, k, mt["nu_sigma_f"]) != 0:
                    raise ValueError("oracle: bad nu_sigma_f")
        for u in spec["universes"]:
            if u["kind"] == "csg":
                uid = L.orc_add_csg_universe(m.h)
                for c in u["cells"]:
                    hs = np.asarray(c["hs"], dtype=np.int32)
                    if "material" in c:
                        fk, f, tr = 0, c["material"], None
                    else:
                        fk, f = 1, c["fill"]
                        tr = np.asarray(c.get("translation", [0.0, 0.0, 0.0]), dtype=np.float64)
                    r = L.orc_add_cell(m.h, uid, _p(hs), len(hs), fk, f,
                                       _p(tr) if tr is not None else None)
                    assert r >= 0
            elif u["kind"] == "rect" and "edges" in u:
                e = np.asarray([v for ax in u["edges"] for v in ax], dtype=np.float64)
                ne = np.asarray([len(ax) for ax in u["edges"]], dtype=np.int32)
                fl = np.asarray(u["fill"], dtype=np.int32)
                if L.orc_add_rect_edges(m.h, _p(e), _p(ne), _p(fl), u["outer"]) < 0:
                    raise ValueError("oracle: bad rect edges")
            elif u["kind"] == "rect":
                ll = np.asarray(u["ll"], dtype=np.float64)
                p = np.asarray(u["pitch"], dtype=np.float64)
                sh = np.asarray(u["shape"], dtype=np.int32)
                fl = np.asarray(u["fill"], dtype=np.int32)
                L.orc_add_rect(m.h, _p(ll), _p(p), _p(sh), _p(fl), u["outer"])
            else:
                cen = np.asarray(u["center"], dtype=np.float64)
                fl = np.asarray(u["fill"], dtype=np.int32)
                L.orc_add_hex(m.h, 0 if u["orient"] == "pointy" else 1, _p(cen), u["pitch"],
                              u["rings"], u["z_lower"], u["z_pitch"], u["nz"], _p(fl), u["outer"])
        L.orc_set_root(m.h, spec["root"])
        m.mesh_shape = None
        if spec.get("mesh"):
            me = spec["mesh"]
            lo, hi = np.asarray(me["lo"], dtype=np.float64), np.asarray(me["hi"], dtype=np.float64)
            sh = np.asarray(me["shape"], dtype=np.int32)
            if L.orc_set_mesh(m.h, _p(lo), _p(hi), _p(sh)) != 0:
                raise ValueError("oracle: bad mesh")
            m.mesh_shape = tuple(int(v) for v in sh)
        rc = L.orc_finalize(m.h)
        if rc != 0:
            raise ValueError(f"oracle finalize failed: {rc}")
        m.n_mc = L.orc_n_material_cells(m.h)
        m.out_len = L.orc_out_len(m.h)
        m.max_depth = L.orc_max_depth(m.h)
        ids = np.zeros(m.n_mc, dtype=np.int32)
        L.orc_material_cell_ids(m.h, _p(ids))
        m.mc_cell = ids
        return m

    # ------------------------------------------------------------------ runs
    def run(self, n: int, seed: int = 240613849, pid_begin: int = 0, lo=None, hi=None,
            max_segments: int = 1_000_000, threads: int | None = None, pflags: bool = False,
            trace_cap: int = 0, states: np.ndarray | None = None, mesh: bool = False,
            instances: bool = False, bank: bool = False, per_history: bool = False):
        """Track particles [pid_begin, pid_begin+n).  Returns dict with out, counters, ...
        mesh=True (model spec with a "mesh"): res["mesh"] = per-voxel track length, x fastest.
        instances=True: res["inst"] = track length per material-cell instance (reading D1).
        bank=True: res["bank"] [n, max_sites, 3] fission sites, res["bank_n"] sites per history (F1)."""
        if threads is None:
            threads = len(os.sched_getaffinity(0))
        out = np.zeros(self.out_len)
        pf = np.zeros(max(n, 1), dtype=np.uint8) if pflags else None
        tr = np.zeros(max(trace_cap, 1), dtype=TRACE_DTYPE) if trace_cap else None
        tcount = np.zeros(1, dtype=np.uint64)
        ev = np.zeros(8, dtype=np.uint64)
        mo = None
        if mesh:
            assert self.mesh_shape is not None, "model has no mesh"
            mo = np.zeros(int(np.prod(self.mesh_shape)))
        io = np.zeros(max(self.n_instances(), 1)) if instances else None
        ms = self.L.orc_max_sites(self.h)
        bk = np.zeros((max(n, 1), ms, 3)) if bank else None
        bn = np.zeros(max(n, 1), dtype=np.uint8) if bank else None
        bargs = (_p(bk), _p(bn)) if bank else (None, None)
        hn = np.zeros(max(n, 1), dtype=np.uint32) if per_history else None
        ht = np.zeros(max(n, 1), dtype=np.uint8) if per_history else None
        bargs = bargs + ((_p(hn), _p(ht)) if per_history else (None, None))
        if states is None:
            src = self.spec["source"]
            lo = np.asarray(src["lo"] if lo is None else lo, dtype=np.float64)
            hi = np.asarray(src["hi"] if hi is None else hi, dtype=np.float64)
            rc = self.L.orc_run(self.h, seed, pid_begin, n, _p(lo), _p(hi), max_segments, threads,
                                _p(out), _p(pf) if pf is not None else None,
                                _p(tr) if tr is not None else None, trace_cap, _p(tcount), _p(ev),
                                _p(mo) if mo is not None else None, _p(io) if io is not None else None,
                                *bargs)
        else:
            st = np.ascontiguousarray(states, dtype=np.float64)
            assert st.shape == (6, n)
            rc = self.L.orc_run_states(self.h, seed, pid_begin, n, _p(st), max_segments, threads,
                                       _p(out), _p(pf) if pf is not None else None,
                                       _p(tr) if tr is not None else None, trace_cap, _p(tcount),
                                       _p(ev), _p(mo) if mo is not None else None,
                                       _p(io) if io is not None else None, *bargs)
        assert rc == 0
        res = self.unpack(out)
        res["evals"] = {k: int(ev[i]) for i, k in enumerate(EVAL_KINDS)}
        if mo is not None:
            res["mesh"] = mo
        if io is not None:
            res["inst"] = io[:self.n_instances()]
        if bank:
            res["bank"], res["bank_n"] = bk[:n], bn[:n]
        if pf is not None:
            res["pflags"] = pf[:n]
        if per_history:
            res["pnseg"], res["pterm"] = hn[:n], ht[:n]
        if tr is not None:
            cnt = int(tcount[0])
            assert cnt <= trace_cap, f"trace overflow {cnt} > {trace_cap}"
            t = tr[:cnt]
            res["trace"] = np.sort(t, order=["pid", "seg", "terminal"])
        return res

    def max_sites(self) -> int:
        return int(self.L.orc_max_sites(self.h))

    def fission_source(self, bank: np.ndarray, bank_n: np.ndarray, seed: int, cycle: int, n_next: int):
        """F1: next cycle's birth states [6, n_next] drawn from the bank; returns (states, M)."""
        bank = np.ascontiguousarray(bank, dtype=np.float64)
        bank_n = np.ascontiguousarray(bank_n, dtype=np.uint8)
        st = np.zeros((6, max(n_next, 1)))
        M = self.L.orc_fission_source(self.h, _p(bank), _p(bank_n), len(bank_n), seed, cycle, n_next, _p(st))
        return st[:, :n_next], int(M)

    @staticmethod
    def bank_sites(bank: np.ndarray, bank_n: np.ndarray) -> np.ndarray:
        """Flat (history, site)-ordered list of banked sites [M, 3] (test helper)."""
        return np.concatenate([bank[h, :bank_n[h]] for h in range(len(bank_n))] + [np.zeros((0, 3))])

    def source_from_sites(self, sites: np.ndarray, seed: int, cycle: int, j_begin: int, n_next: int):
        """F1 multi-rank form: particles j_begin .. j_begin + n_next - 1 from a flat site list."""
        sites = np.ascontiguousarray(sites, dtype=np.float64).reshape(-1, 3)
        st = np.zeros((6, max(n_next, 1)))
        self.L.orc_source_from_sites(_p(sites), len(sites), seed, cycle, j_begin, n_next, _p(st))
        return st[:, :n_next]

    def power_iteration(self, n: int, cycles: int, seed: int = 240613849):
        """F1 power iteration (Alg. 1): cycle 0 born in the source box, then from the bank; histories
        of cycle c use pids [c << 32, (c << 32) + n).  Returns the k estimate of every cycle."""
        ks, states = [], None
        for c in range(cycles):
            res = self.run(n, seed=seed, pid_begin=c << 32, bank=True, states=states)
            ks.append(int(res["bank_n"].sum()) / n)
            states, M = self.fission_source(res["bank"], res["bank_n"], seed, c, n)
            if M == 0:
                raise RuntimeError("fission source collapsed (no sites banked)")
        return ks

    def n_instances(self) -> int:
        """Material-cell instances in the model (reading D1)."""
        return int(self.L.orc_n_instances(self.h))

    def instance_cells(self) -> np.ndarray:
        """Material-cell index of every instance, by explicit depth-first enumeration (D1)."""
        out = np.zeros(max(self.n_instances(), 1), dtype=np.int32)
        self.L.orc_instance_cells(self.h, _p(out))
        return out[:self.n_instances()]

    def unpack(self, out: np.ndarray) -> dict:
        n = self.n_mc
        return {"out": out, "len": out[:n], "exits": out[n:2 * n],
                "counters": {k: int(out[2 * n + i]) for i, k in enumerate(COUNTERS)}}

    def falg(self, res: dict) -> float:
        """Algorithmic fp64 flops per segment from evaluation counts."""
        seg = res["counters"]["segments"]
        return sum(EVAL_FLOPS[k] * v for k, v in res["evals"].items()) / max(seg, 1)

    # ------------------------------------------------------------------ queries
    def find_cells(self, xyz: np.ndarray):
        xyz = np.ascontiguousarray(xyz, dtype=np.float64)
        n = xyz.shape[1]
        cells = np.zeros(n, dtype=np.int32)
        fl = np.zeros(n, dtype=np.uint8)
        self.L.orc_find_cells(self.h, _p(xyz), n, _p(cells), _p(fl))
        return cells, fl

    def count_containing(self, uid: int, r) -> int:
        r = np.asarray(r, dtype=np.float64)
        return self.L.orc_count_containing(self.h, uid, _p(r))

    def surface_distance(self, sid: int, sense_pos: bool, r, om, onsurf: bool = False) -> float:
        r = np.asarray(r, dtype=np.float64)
        om = np.asarray(om, dtype=np.float64)
        return self.L.orc_surface_distance(self.h, sid, int(sense_pos), int(onsurf), _p(r), _p(om))

    def surface_f(self, sid: int, r) -> float:
        r = np.asarray(r, dtype=np.float64)
        return self.L.orc_surface_f(self.h, sid, _p(r))

    def locate_array(self, uid: int, rl):
        rl = np.asarray(rl, dtype=np.float64)
        ijk = np.zeros(3, dtype=np.int32)
        d = np.zeros(1, dtype=np.int32)
        t = np.zeros(3)
        fl = np.zeros(1, dtype=np.int32)
        ok = self.L.orc_locate_array(self.h, uid, _p(rl), _p(ijk), _p(d), _p(t), _p(fl))
        return bool(ok), tuple(int(v) for v in ijk), int(d[0]), t, int(fl[0])

    def hex_owns(self, uid: int, q: int, r: int, rl) -> bool:
        rl = np.asarray(rl, dtype=np.float64)
        return bool(self.L.orc_hex_owns(self.h, uid, q, r, _p(rl)))

    def cell_material(self, cell: int) -> int:
        return self.L.orc_cell_material(self.h, cell)
