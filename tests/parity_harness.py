"""SURVEY §8(c)4 per-cell parity with flagged-history exclusion (shared by the GPU parity tests).

1. both sides track the batch and return per-history O16 flags;
2. U = the union of the pids either side flagged;
3. U is re-run alone on both sides (a walk is a pure function of (seed, pid), O17), in contiguous
   pid runs;
4. U's contributions are subtracted, and the remaining totals are compared: counters and exits
   exactly, track lengths within 1e-9 relative (the contract's per-cell tolerance).
"""
from __future__ import annotations

import numpy as np

LEN_RTOL = 1e-9


def runs_of(idx: np.ndarray):
    """Contiguous runs [(start, length)] of a sorted index array."""
    out = []
    if len(idx) == 0:
        return out
    s = p = int(idx[0])
    for v in idx[1:]:
        v = int(v)
        if v != p + 1:
            out.append((s, p - s + 1))
            s = v
        p = v
    out.append((s, p - s + 1))
    return out


def gpu_side(m, seed, gpu_kw=None, states=None):
    """(n, pid_begin[, states slice]) -> (packed out, pflags) through nt_track / nt_track_states."""
    import torch
    kw = dict(gpu_kw or {})

    def run(n, pid_begin, lo_idx=0):
        st = None
        if states is not None:
            st = torch.tensor(states[:, lo_idx:lo_idx + n], dtype=torch.float64, device="cuda").contiguous()
        res = m.track(n, seed=seed, pid_begin=pid_begin, pflags=True, states=st, **kw)
        torch.cuda.synchronize()
        return res["out"].cpu().numpy().copy(), res["pflags"].cpu().numpy()[:n].copy()
    return run


def oracle_side(om, seed, states=None, **okw):
    def run(n, pid_begin, lo_idx=0):
        st = None if states is None else np.ascontiguousarray(states[:, lo_idx:lo_idx + n])
        r = om.run(n, seed=seed, pid_begin=pid_begin, pflags=True, states=st, **okw)
        return r["out"].copy(), r["pflags"].copy()
    return run


def compare_excluding_flagged(gpu_run, orc_run, n_mc: int, n: int, pid_begin: int = 0,
                              len_rtol: float = LEN_RTOL):
    """Run both sides, exclude the union of flagged pids, compare.  Returns a report dict."""
    g, gpf = gpu_run(n, pid_begin)
    o, opf = orc_run(n, pid_begin)
    U = np.nonzero((gpf != 0) | (opf != 0))[0]
    gU = np.zeros_like(g)
    oU = np.zeros_like(o)
    for s, k in runs_of(U):
        gg, gf = gpu_run(k, pid_begin + s, s)
        oo, of = orc_run(k, pid_begin + s, s)
        # a walk is a pure function of (seed, pid): re-run alone, every pid flags as it did
        assert np.array_equal(gf, gpf[s:s + k]) and np.array_equal(of, opf[s:s + k])
        gU += gg
        oU += oo
    ge, oe = g - gU, o - oU
    nc = len(g) - 2 * n_mc
    gc, oc = ge[2 * n_mc:], oe[2 * n_mc:]
    assert np.array_equal(gc, oc), ("counters after exclusion", gc, oc)
    assert np.array_equal(ge[n_mc:2 * n_mc], oe[n_mc:2 * n_mc]), "exits after exclusion"
    gl, ol = ge[:n_mc], oe[:n_mc]
    assert np.all(np.abs(gl - ol) <= len_rtol * np.abs(ol) + 1e-300), ("len after exclusion", gl, ol)
    return {"n": n, "flagged_gpu": int((gpf != 0).sum()), "flagged_oracle": int((opf != 0).sum()),
            "union": int(len(U)), "flags_equal": bool(np.array_equal(gpf, opf)), "n_counters": nc,
            "max_len_rel": float(np.max(np.abs(gl - ol) / np.maximum(np.abs(ol), 1e-300))),
            "gpu": g, "oracle": o, "gpu_pflags": gpf, "oracle_pflags": opf}
