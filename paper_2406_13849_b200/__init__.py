"""nestrack: B200-native nested-geometry Monte Carlo tracking (arXiv 2406.13849 hot path).

Thin Python binding over the C ABI of ``libnestrack.so`` (include/nestrack.h).  This module
only marshals arguments: every step of the tracking path runs in the library's CUDA kernels.
PyTorch provides device memory, streams and process groups.  There is no CPU fallback: if the
library is missing, importing :func:`lib` raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("NESTRACK_LIB", os.path.join(HERE, "libnestrack.so"))   # override: tuning builds

KIND = {"PX": 0, "PY": 1, "PZ": 2, "PLANE": 3, "CZ": 4, "SPHERE": 5}
BC = {"none": 0, "vacuum": 1, "reflect": 2}
TRACKER = {"generic": 0, "rect": 1}
NT_TRACE = 1
NT_HISTORY = 2
NT_WARPQ = 4
NT_DP = 8
NT_ROUNDS = 16
# "block": block queues as shared-memory rings, no rounds / barriers (default); "rounds": the
# round-based form with one block barrier per round; "dp" / "dp-rounds": dynamic-polymorphism
# dispatch (virtual tracker calls) in either form
SCHEDULERS = {"block": 0, "event": 0, "rounds": NT_ROUNDS, "warp": NT_WARPQ, "history": NT_HISTORY,
              "dp": NT_DP, "dp-rounds": NT_DP | NT_ROUNDS}
COUNTERS = ["particles", "segments", "crossings", "reflections", "leaks", "collisions",
            "absorptions", "lost", "capped", "flagged"] + [f"cross_l{i}" for i in range(8)]
NC = len(COUNTERS)
STATUS = {0: "NT_OK", -1: "NT_E_ARG", -2: "NT_E_ID", -3: "NT_E_ORDER", -4: "NT_E_GEOMETRY",
          -5: "NT_E_UNSUPPORTED", -6: "NT_E_CUDA", -7: "NT_E_NOMEM"}

TRACE_DTYPE = np.dtype([("pid", "<u8"), ("s", "<f8"), ("seg", "<u4"), ("cell_before", "<i4"),
                        ("cell_after", "<i4"), ("j", "<i4"), ("kind", "u1"), ("level", "i1"),
                        ("terminal", "u1"), ("pad", "u1"), ("flags", "<u4")])


class NtError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class BuildOpts(C.Structure):
    _fields_ = [("device", C.c_int32), ("bih_max_leaf", C.c_int32), ("pseudo_array", C.c_int32),
                ("reserved", C.c_int32), ("sah_ct", C.c_double), ("sah_ci", C.c_double)]


class ModelInfo(C.Structure):
    _fields_ = [("n_surfaces", C.c_int32), ("n_cells", C.c_int32), ("n_material_cells", C.c_int32),
                ("n_universes", C.c_int32), ("max_depth", C.c_int32),
                ("rect_specialisable", C.c_int32), ("rect_levels", C.c_int32),
                ("n_bih_nodes", C.c_int32), ("out_len", C.c_int64), ("device_bytes", C.c_size_t),
                ("mesh_bins", C.c_int64), ("n_instances", C.c_int64), ("max_sites", C.c_int32)]


class Run(C.Structure):
    _fields_ = [("seed", C.c_uint64), ("pid_begin", C.c_uint64), ("n", C.c_uint64),
                ("src_lo", C.c_double * 3), ("src_hi", C.c_double * 3),
                ("max_segments", C.c_uint64), ("tracker", C.c_int32), ("flags", C.c_uint32),
                ("block_dim", C.c_int32), ("blocks_per_sm", C.c_int32)]


class Outputs(C.Structure):
    _fields_ = [("out", C.c_void_p), ("pflags", C.c_void_p), ("pnseg", C.c_void_p),
                ("pterm", C.c_void_p), ("trace", C.c_void_p),
                ("trace_cap", C.c_uint64), ("trace_count", C.c_void_p), ("mesh", C.c_void_p),
                ("inst", C.c_void_p), ("bank", C.c_void_p), ("bank_n", C.c_void_p)]


_lib = None

SYMBOLS = ["nt_last_error", "nt_abi_version", "nt_model_create", "nt_model_destroy", "nt_add_surface",
           "nt_add_material", "nt_add_csg_universe", "nt_add_cell", "nt_add_rect_array", "nt_add_rect_edges",
           "nt_add_hex_array", "nt_set_root", "nt_set_mesh", "nt_build_opts_default", "nt_finalize",
           "nt_model_info_get", "nt_material_cell_ids", "nt_instance_cells", "nt_set_fission",
           "nt_fission_source", "nt_bank_compact", "nt_source_from_sites", "nt_bih_info", "nt_track",
           "nt_track_states", "nt_track_host", "nt_find_cells", "nt_last_launch_count",
           "nt_selftest_arith"]


def lib():
    """Load libnestrack.so (raises if it was not built: there is no fallback path)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = C.CDLL(LIB_PATH)
        vp, i32, u64, dp = C.c_void_p, C.c_int32, C.c_uint64, C.c_void_p
        L.nt_last_error.restype = C.c_char_p
        L.nt_model_create.argtypes = [C.POINTER(vp)]
        L.nt_model_destroy.argtypes = [vp]
        L.nt_add_surface.argtypes = [vp, i32, dp, i32, C.POINTER(i32)]
        L.nt_add_material.argtypes = [vp, C.c_double, C.c_double, C.POINTER(i32)]
        L.nt_add_csg_universe.argtypes = [vp, C.POINTER(i32)]
        L.nt_add_cell.argtypes = [vp, i32, dp, i32, i32, i32, dp, C.POINTER(i32)]
        L.nt_add_rect_array.argtypes = [vp, dp, dp, dp, dp, i32, C.POINTER(i32)]
        L.nt_add_rect_edges.argtypes = [vp, dp, dp, dp, i32, C.POINTER(i32)]
        L.nt_add_hex_array.argtypes = [vp, i32, dp, C.c_double, i32, C.c_double, C.c_double, i32, dp,
                                       i32, C.POINTER(i32)]
        L.nt_set_root.argtypes = [vp, i32]
        L.nt_set_mesh.argtypes = [vp, dp, dp, dp]
        L.nt_instance_cells.argtypes = [vp, dp, C.c_int64]
        L.nt_set_fission.argtypes = [vp, i32, C.c_double]
        L.nt_bank_compact.argtypes = [vp, vp, vp, C.c_uint64, vp, C.POINTER(C.c_uint64), vp]
        L.nt_source_from_sites.argtypes = [vp, vp, C.c_uint64, C.c_uint64, C.c_uint32, C.c_uint64, C.c_uint64, vp, vp]
        L.nt_fission_source.argtypes = [vp, vp, vp, C.c_uint64, C.c_uint64, C.c_uint32, C.c_uint64, vp,
                                        C.POINTER(C.c_uint64), vp]
        L.nt_build_opts_default.argtypes = [C.POINTER(BuildOpts)]
        L.nt_finalize.argtypes = [vp, C.POINTER(BuildOpts)]
        L.nt_model_info_get.argtypes = [vp, C.POINTER(ModelInfo)]
        L.nt_material_cell_ids.argtypes = [vp, dp, i32]
        L.nt_bih_info.argtypes = [vp, i32, C.POINTER(i32), C.POINTER(i32), dp, i32, C.POINTER(i32)]
        L.nt_track.argtypes = [vp, C.POINTER(Run), C.POINTER(Outputs), vp]
        L.nt_track_states.argtypes = [vp, C.POINTER(Run), dp, C.POINTER(Outputs), vp]
        L.nt_track_host.argtypes = [vp, C.POINTER(Run), dp, vp]
        L.nt_find_cells.argtypes = [vp, dp, u64, dp, dp, vp]
        L.nt_last_launch_count.argtypes = [vp]
        L.nt_selftest_arith.argtypes = [u64, u64, dp]
        _lib = L
    return _lib


def _check(st: int):
    if st != 0:
        raise NtError(st, lib().nt_last_error().decode())


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _stream_handle(stream):
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return C.c_void_p(stream.cuda_stream)


class Model:
    """A nested CSG model: builder calls (nt_add_*), finalize, then tracking on one GPU."""

    def __init__(self):
        self.L = lib()
        self.h = C.c_void_p()
        _check(self.L.nt_model_create(C.byref(self.h)))
        self.info = None
        self.spec = None

    def __del__(self):
        try:
            self.L.nt_model_destroy(self.h)
        except Exception:
            pass

    # ---------------------------------------------------------------- builder
    def add_surface(self, kind: str, coef, bc: str = "none") -> int:
        c = np.zeros(4)
        c[:len(coef)] = coef
        i = C.c_int32()
        _check(self.L.nt_add_surface(self.h, KIND[kind], _p(c), BC[bc], C.byref(i)))
        return i.value

    def add_material(self, sigma_t: float, sigma_a: float) -> int:
        i = C.c_int32()
        _check(self.L.nt_add_material(self.h, sigma_t, sigma_a, C.byref(i)))
        return i.value

    def set_fission(self, mat: int, nu_sigma_f: float):
        """One-group nu Sigma_f of material `mat` (reading F1; validated at finalize)."""
        _check(self.L.nt_set_fission(self.h, mat, nu_sigma_f))

    def add_csg_universe(self) -> int:
        i = C.c_int32()
        _check(self.L.nt_add_csg_universe(self.h, C.byref(i)))
        return i.value

    def add_cell(self, uid: int, halfspaces, material: int | None = None, fill: int | None = None,
                 translation=None) -> int:
        hs = np.asarray(halfspaces, dtype=np.int32)
        tr = None if translation is None else np.asarray(translation, dtype=np.float64)
        fk, f = (0, material) if material is not None else (1, fill)
        i = C.c_int32()
        _check(self.L.nt_add_cell(self.h, uid, _p(hs) if len(hs) else None, len(hs), fk, f,
                                  _p(tr) if tr is not None else None, C.byref(i)))
        return i.value

    def add_rect_array(self, ll, pitch, shape, fill, outer: int = -1) -> int:
        a = np.asarray(ll, dtype=np.float64)
        p = np.asarray(pitch, dtype=np.float64)
        s = np.asarray(shape, dtype=np.int32)
        f = np.asarray(fill, dtype=np.int32)
        i = C.c_int32()
        _check(self.L.nt_add_rect_array(self.h, _p(a), _p(p), _p(s), _p(f), outer, C.byref(i)))
        return i.value

    def add_rect_edges(self, edges, fill, outer: int = -1) -> int:
        """Non-uniform rect array: edges = [ex, ey, ez] (ez empty: 2-D)."""
        e = np.asarray([v for ax in edges for v in ax], dtype=np.float64)
        ne = np.asarray([len(ax) for ax in edges], dtype=np.int32)
        f = np.asarray(fill, dtype=np.int32)
        i = C.c_int32()
        _check(self.L.nt_add_rect_edges(self.h, _p(e), _p(ne), _p(f), outer, C.byref(i)))
        return i.value

    def add_hex_array(self, orient: str, center, pitch: float, rings: int, fill, outer: int = -1,
                      z_lower: float = 0.0, z_pitch: float = 0.0, nz: int = 0) -> int:
        c = np.asarray(center, dtype=np.float64)
        f = np.asarray(fill, dtype=np.int32)
        i = C.c_int32()
        _check(self.L.nt_add_hex_array(self.h, 0 if orient == "pointy" else 1, _p(c), pitch, rings,
                                       z_lower, z_pitch, nz, _p(f), outer, C.byref(i)))
        return i.value

    def set_root(self, uid: int):
        _check(self.L.nt_set_root(self.h, uid))

    def set_mesh(self, lo, hi, shape):
        """Superimposed Cartesian mesh for the track-length mesh tally (reading M1)."""
        lo_, hi_ = np.asarray(lo, dtype=np.float64), np.asarray(hi, dtype=np.float64)
        sh = np.asarray(shape, dtype=np.int32)
        _check(self.L.nt_set_mesh(self.h, _p(lo_), _p(hi_), _p(sh)))

    def finalize(self, device: int = 0, pseudo_array: bool = False, bih_max_leaf: int = 4):
        o = BuildOpts()
        self.L.nt_build_opts_default(C.byref(o))
        o.device = device
        o.pseudo_array = int(pseudo_array)
        o.bih_max_leaf = bih_max_leaf
        _check(self.L.nt_finalize(self.h, C.byref(o)))
        inf = ModelInfo()
        _check(self.L.nt_model_info_get(self.h, C.byref(inf)))
        self.info = {k: getattr(inf, k) for k, _ in ModelInfo._fields_}
        self.device = device
        self.n_mc = inf.n_material_cells
        self.out_len = inf.out_len
        ids = np.zeros(max(self.n_mc, 1), dtype=np.int32)
        _check(self.L.nt_material_cell_ids(self.h, _p(ids), self.n_mc))
        self.mc_cell = ids[:self.n_mc]
        return self

    @classmethod
    def from_spec(cls, spec: dict, device: int = 0, pseudo_array: bool = False,
                  bih_max_leaf: int = 4) -> "Model":
        """Build from a workloads spec dict (surfaces, materials, universes in list order)."""
        m = cls()
        m.spec = spec
        for s in spec["surfaces"]:
            m.add_surface(s["kind"], s["coef"], s["bc"])
        for mt in spec["materials"]:
            k = m.add_material(mt["sigma_t"], mt["sigma_a"])
            if mt.get("nu_sigma_f", 0.0):
                m.set_fission(k, mt["nu_sigma_f"])
        for u in spec["universes"]:
            if u["kind"] == "csg":
                uid = m.add_csg_universe()
                for c in u["cells"]:
                    if "material" in c:
                        m.add_cell(uid, c["hs"], material=c["material"])
                    else:
                        m.add_cell(uid, c["hs"], fill=c["fill"], translation=c.get("translation"))
            elif u["kind"] == "rect" and "edges" in u:
                m.add_rect_edges(u["edges"], u["fill"], u["outer"])
            elif u["kind"] == "rect":
                m.add_rect_array(u["ll"], u["pitch"], u["shape"], u["fill"], u["outer"])
            else:
                m.add_hex_array(u["orient"], u["center"], u["pitch"], u["rings"], u["fill"], u["outer"],
                                u["z_lower"], u["z_pitch"], u["nz"])
        m.set_root(spec["root"])
        if spec.get("mesh"):
            m.set_mesh(spec["mesh"]["lo"], spec["mesh"]["hi"], spec["mesh"]["shape"])
        return m.finalize(device=device, pseudo_array=pseudo_array, bih_max_leaf=bih_max_leaf)

    def bih_info(self, uid: int):
        nn, dep, cnt = C.c_int32(), C.c_int32(), C.c_int32()
        _check(self.L.nt_bih_info(self.h, uid, C.byref(nn), C.byref(dep), None, 0, C.byref(cnt)))
        cells = np.zeros(max(cnt.value, 1), dtype=np.int32)
        _check(self.L.nt_bih_info(self.h, uid, C.byref(nn), C.byref(dep), _p(cells), cnt.value,
                                  C.byref(cnt)))
        return {"n_nodes": nn.value, "depth": dep.value, "leaf_cells": cells[:cnt.value]}

    # ---------------------------------------------------------------- tracking
    def make_run(self, n: int, seed: int, pid_begin: int = 0, lo=None, hi=None, max_segments: int = 0,
                 tracker: str = "generic", trace: bool = False, block_dim: int = 0,
                 blocks_per_sm: int = 0, scheduler: str = "block") -> Run:
        r = Run()
        r.seed, r.pid_begin, r.n = seed, pid_begin, n
        src = (self.spec or {}).get("source", {"lo": [0, 0, 0], "hi": [0, 0, 0]})
        lo = src["lo"] if lo is None else lo
        hi = src["hi"] if hi is None else hi
        for a in range(3):
            r.src_lo[a], r.src_hi[a] = lo[a], hi[a]
        r.max_segments = max_segments
        r.tracker = TRACKER[tracker]
        assert scheduler in SCHEDULERS
        r.flags = (NT_TRACE if trace else 0) | SCHEDULERS[scheduler]
        r.block_dim, r.blocks_per_sm = block_dim, blocks_per_sm
        return r

    def track(self, n: int, seed: int = 240613849, pid_begin: int = 0, lo=None, hi=None,
              max_segments: int = 0, tracker: str = "generic", pflags: bool = False,
              trace_cap: int = 0, states=None, out=None, stream=None, block_dim: int = 0,
              blocks_per_sm: int = 0, per_history: bool = False, scheduler: str = "block", mesh=None,
              instances=None, bank: bool = False):
        """Track histories [pid_begin, pid_begin+n) on this model's GPU (async on `stream`).
        Returns a dict of device tensors: out (accumulated), pflags, trace, trace_count."""
        import torch
        dev = torch.device("cuda", self.device)
        if out is None:
            out = torch.zeros(self.out_len, dtype=torch.float64, device=dev)
        res = {"out": out}
        o = Outputs()
        o.out = out.data_ptr()
        if pflags:
            pf = torch.zeros(max(n, 1), dtype=torch.uint8, device=dev)
            o.pflags = pf.data_ptr()
            res["pflags"] = pf
        if per_history:
            ps = torch.zeros(max(n, 1), dtype=torch.int32, device=dev)
            pt = torch.zeros(max(n, 1), dtype=torch.uint8, device=dev)
            o.pnseg, o.pterm = ps.data_ptr(), pt.data_ptr()
            res["pnseg"], res["pterm"] = ps, pt
        if trace_cap:
            tr = torch.zeros(trace_cap * TRACE_DTYPE.itemsize, dtype=torch.uint8, device=dev)
            tc = torch.zeros(1, dtype=torch.int64, device=dev)
            o.trace, o.trace_cap, o.trace_count = tr.data_ptr(), trace_cap, tc.data_ptr()
            res["trace"], res["trace_count"] = tr, tc
        if mesh is not None:                       # True: fresh zeroed tensor; or a caller tensor
            if mesh is True:
                mesh = torch.zeros(max(self.info["mesh_bins"], 1), dtype=torch.float64, device=dev)
            assert mesh.dtype == torch.float64 and mesh.is_cuda and mesh.numel() >= self.info["mesh_bins"] > 0
            o.mesh = mesh.data_ptr()
            res["mesh"] = mesh
        if instances is not None:                  # per-instance tally (reading D1)
            if instances is True:
                instances = torch.zeros(max(self.info["n_instances"], 1), dtype=torch.float64, device=dev)
            assert instances.dtype == torch.float64 and instances.is_cuda
            assert instances.numel() >= self.info["n_instances"] > 0
            o.inst = instances.data_ptr()
            res["inst"] = instances
        if bank:                                   # fission bank (reading F1)
            ms = self.info["max_sites"]
            bk = torch.empty(max(n, 1) * ms * 3, dtype=torch.float64, device=dev)
            bn = torch.empty(max(n, 1), dtype=torch.uint8, device=dev)
            o.bank, o.bank_n = bk.data_ptr(), bn.data_ptr()
            res["bank"], res["bank_n"] = bk, bn
        run = self.make_run(n, seed, pid_begin, lo, hi, max_segments, tracker, bool(trace_cap),
                            block_dim, blocks_per_sm, scheduler)
        sh = _stream_handle(stream)
        if states is not None:
            assert states.dtype == torch.float64 and states.is_cuda and tuple(states.shape) == (6, n)
            states = states.contiguous()
            res["_states"] = states
            _check(self.L.nt_track_states(self.h, C.byref(run), C.c_void_p(states.data_ptr()),
                                          C.byref(o), sh))
        else:
            _check(self.L.nt_track(self.h, C.byref(run), C.byref(o), sh))
        return res

    def track_host(self, n: int, seed: int = 240613849, pid_begin: int = 0, lo=None, hi=None,
                   max_segments: int = 0, tracker: str = "generic", out: np.ndarray | None = None,
                   stream=None, block_dim: int = 0, blocks_per_sm: int = 0,
                   scheduler: str = "block") -> np.ndarray:
        """End-to-end call with a HOST output buffer (synchronous)."""
        if out is None:
            out = np.zeros(self.out_len)
        run = self.make_run(n, seed, pid_begin, lo, hi, max_segments, tracker, False, block_dim,
                            blocks_per_sm, scheduler)
        _check(self.L.nt_track_host(self.h, C.byref(run), _p(out), _stream_handle(stream)))
        return out

    def find_cells(self, xyz, stream=None):
        import torch
        xyz = xyz.contiguous()
        n = xyz.shape[1]
        cell = torch.empty(n, dtype=torch.int32, device=xyz.device)
        fl = torch.empty(n, dtype=torch.uint8, device=xyz.device)
        _check(self.L.nt_find_cells(self.h, C.c_void_p(xyz.data_ptr()), n, C.c_void_p(cell.data_ptr()),
                                    C.c_void_p(fl.data_ptr()), _stream_handle(stream)))
        return cell, fl

    def fission_source(self, bank, bank_n, n_prev: int, seed: int, cycle: int, n_next: int, stream=None):
        """F1: next cycle's birth states [6, n_next] (device) drawn from a bank; returns (states, M)."""
        import torch
        st = torch.empty((6, max(n_next, 1)), dtype=torch.float64, device=torch.device("cuda", self.device))
        M = C.c_uint64()
        _check(self.L.nt_fission_source(self.h, C.c_void_p(bank.data_ptr()), C.c_void_p(bank_n.data_ptr()),
                                        n_prev, seed, cycle, n_next, C.c_void_p(st.data_ptr()), C.byref(M),
                                        _stream_handle(stream)))
        return st[:, :n_next], int(M.value)

    def power_iteration(self, n: int, cycles: int, seed: int = 240613849, scheduler: str = "block"):
        """F1 power iteration (Alg. 1) on the device: cycle 0 born in the source box, later cycles
        from the previous bank; cycle c uses pids [c << 32, (c << 32) + n).  Returns per-cycle k."""
        import torch
        ks, states = [], None
        for c in range(cycles):
            res = self.track(n, seed=seed, pid_begin=c << 32, bank=True, states=states, scheduler=scheduler)
            nb = int(res["bank_n"][:n].sum().item())
            ks.append(nb / n)
            states, M = self.fission_source(res["bank"], res["bank_n"], n, seed, c, n)
            if M == 0:
                raise RuntimeError("fission source collapsed (no sites banked)")
            states = states.contiguous()
        return ks

    def instance_cells(self) -> np.ndarray:
        """Material-cell bin of every material-cell instance (reading D1)."""
        n = self.info["n_instances"]
        out = np.zeros(max(n, 1), dtype=np.int32)
        _check(self.L.nt_instance_cells(self.h, _p(out), n))
        return out[:n]

    def last_launch_count(self) -> int:
        return self.L.nt_last_launch_count(self.h)

    # ---------------------------------------------------------------- results
    def unpack(self, out) -> dict:
        o = out.detach().cpu().numpy() if hasattr(out, "detach") else np.asarray(out)
        n = self.n_mc
        return {"out": o, "len": o[:n], "exits": o[n:2 * n],
                "counters": {k: int(o[2 * n + i]) for i, k in enumerate(COUNTERS)}}

    @staticmethod
    def trace_records(res) -> np.ndarray:
        cnt = int(res["trace_count"].item())
        buf = res["trace"].cpu().numpy()
        cap = buf.size // TRACE_DTYPE.itemsize
        assert cnt <= cap, f"trace overflow: {cnt} > {cap}"
        t = buf[:cnt * TRACE_DTYPE.itemsize].view(TRACE_DTYPE)
        return np.sort(t, order=["pid", "seg", "terminal"])


def selftest_arith(n: int = 1 << 26, seed: int = 1):
    """Device check of the kernels' division / sqrt against IEEE: returns (div, sqrt) mismatches."""
    out = np.zeros(2, dtype=np.uint64)
    _check(lib().nt_selftest_arith(n, seed, _p(out)))
    return int(out[0]), int(out[1])


def shard(n_total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous pid shard of rank g of G: [floor(gN/G), floor((g+1)N/G))."""
    b = n_total * rank // world
    e = n_total * (rank + 1) // world
    return b, e - b


def track_distributed(model: Model, n_total: int, seed: int, pid_begin: int = 0, group=None,
                      tracker_fn=None, **kw):
    """Multi-GPU tracking: each rank tracks its contiguous pid shard on its own GPU, then ONE
    all-reduce (sum) of the packed fp64 [len | exits | counters] buffer combines the tallies.
    `tracker_fn(n, pid_begin) -> out tensor` overrides the per-rank tracker (CPU tests)."""
    import torch.distributed as dist
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    b, n = shard(n_total, rank, world)
    if tracker_fn is None:
        out = model.track(n, seed=seed, pid_begin=pid_begin + b, **kw)["out"]
    else:
        out = tracker_fn(n, pid_begin + b)
    if world > 1:
        _all_reduce_sum(out, group)
    return out


def _host_staged(group) -> bool:
    """gloo runs all_gather on host tensors only (and is the backend of the CPU / one-GPU
    multi-rank tests); NCCL takes device tensors directly."""
    import torch.distributed as dist
    return dist.get_backend(group) == "gloo"


def _all_reduce_sum(t, group=None):
    import torch.distributed as dist
    if t.is_cuda and _host_staged(group):
        h = t.cpu()
        dist.all_reduce(h, op=dist.ReduceOp.SUM, group=group)
        t.copy_(h)
    else:
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)


def _all_gather(t, world: int, group=None):
    import torch.distributed as dist
    if t.is_cuda and _host_staged(group):
        h = t.cpu()
        bufs = [h.new_zeros(h.shape) for _ in range(world)]
        dist.all_gather(bufs, h, group=group)
        return [b.to(t.device) for b in bufs]
    bufs = [t.new_zeros(t.shape) for _ in range(world)]
    dist.all_gather(bufs, t, group=group)
    return bufs


def power_iteration_distributed(model: Model, n: int, cycles: int, seed: int = 240613849, group=None,
                                track_fn=None, sample_fn=None, scheduler: str = "block"):
    """Multi-GPU power iteration (reading F1, Alg. 1): every rank tracks n histories per cycle
    (cycle c, rank r: pids (c << 32) + r n ...), compacts its fission bank, and the ranks
    all-gather the site counts and the sites (the cycle's real exchange: the next source is drawn
    from the global bank).  Rank r then draws source particles J = r n .. (r + 1) n - 1 from the
    (rank, history, site)-ordered global list, so the result equals one process tracking all
    world * n histories.  Returns the k estimate of every cycle (the same on every rank).

    track_fn(n, pid_begin, states, cycle) -> (sites [M_r, 3] tensor, M_r) and
    sample_fn(sites, M, cycle, j_begin, n) -> states override the device calls (CPU tests)."""
    import torch
    import torch.distributed as dist
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    if track_fn is None:
        def track_fn(nn, pid0, states, cycle):
            res = model.track(nn, seed=seed, pid_begin=pid0, bank=True, states=states, scheduler=scheduler)
            ms = model.info["max_sites"]
            sites = torch.empty(max(nn * ms, 1) * 3, dtype=torch.float64, device=res["bank"].device)
            M = C.c_uint64()
            _check(model.L.nt_bank_compact(model.h, C.c_void_p(res["bank"].data_ptr()),
                                           C.c_void_p(res["bank_n"].data_ptr()), nn,
                                           C.c_void_p(sites.data_ptr()), C.byref(M),
                                           _stream_handle(None)))
            return sites[:3 * M.value].view(-1, 3), int(M.value)
    if sample_fn is None:
        def sample_fn(sites, M, cycle, j0, nn):
            st = torch.empty((6, max(nn, 1)), dtype=torch.float64, device=sites.device)
            sites = sites.contiguous()
            _check(model.L.nt_source_from_sites(model.h, C.c_void_p(sites.data_ptr()), M, seed, cycle, j0, nn,
                                                C.c_void_p(st.data_ptr()), _stream_handle(None)))
            return st[:, :nn].contiguous()
    ks, states = [], None
    for c in range(cycles):
        sites, Mr = track_fn(n, (c << 32) + rank * n, states, c)
        if world > 1:
            cnt = torch.tensor([Mr], dtype=torch.int64, device=sites.device)
            counts = [int(x.item()) for x in _all_gather(cnt, world, group)]
            pad = max(max(counts), 1)
            buf = torch.zeros((pad, 3), dtype=torch.float64, device=sites.device)
            buf[:Mr] = sites
            bufs = _all_gather(buf, world, group)
            sites = torch.cat([bufs[r][:counts[r]] for r in range(world)])
            M = sum(counts)
        else:
            M = Mr
        ks.append(M / (world * n))
        if M == 0:
            raise RuntimeError("fission source collapsed (no sites banked)")
        states = sample_fn(sites, M, c, rank * n, n)
    return ks
