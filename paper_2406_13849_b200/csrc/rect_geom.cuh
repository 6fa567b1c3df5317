// Rect-specialised tracker (RTK, §3.3 Alg. 9-10) operations on the
// shared-memory universe stack of the event-queue scheduler (event_kernel.cuh, RTK != 0).
//
// Model shape (rect_spec.cpp gates it): root = axis box (BOX) or concentric CZ annuli between a PZ
// pair -> K rect arrays (K = rg.K <= 4) -> concentric-CZ pin.  The code is non-polymorphic: no
// universe-kind dispatch, no BIH, closed-form rect indexing and a linear annulus search, with the
// level loop unrolled to 4 and guarded by the model's K.  The arithmetic is exactly that of the
// history-based RTK (rect_kernel.cuh) and of the generic tracker, so all three are bit-identical.
//
// Stack layout (the generic Stack accessors):
//   level 0      root:  a = annulus (CZ root; 0 = core), u = root universe
//   level 1..K   rect:  u = array universe, a, b, c = tile i, j, k; T = frame
//   level K+1    pin:   u = pin universe, a = pin index, b = annulus; T = frame
// L = K + 2 in the core, 1 in an outer root annulus (its material cell sits at level 0).
// A CSG-level distance key holds the surface id (not a half-space index as in the generic tracker).
#pragma once

NT_DEV_BEGIN

constexpr int kRectMaxK = 4;

// Alg. 9 find_cell from level l0 (0: root; 1..K: rect level whose universe and frame are already in
// the stack; K+1: pin).  fsid >= 0: a CSG crossing at level l0, whose surface takes sense fsense.
template <bool BOX>
__device__ __forceinline__ bool rect_descend(const DevGeom& g, const RectGeom& rg, Stack& st, int l0, int fsid,
                                             int fsense, double rx, double ry, double rz, int& L, int& mc,
                                             uint32_t& flags) {
  const int K = rg.K, KP = K + 1;
  bool ok = true, core = true;
  if (l0 == 0) {
    uint32_t nb = 0;
    int ann = 0;
    if (BOX) {
#pragma unroll
      for (int k = 0; k < 6; ++k) {
        const int sid = rg.box_sid[k];
        int s;
        if (sid == fsid) {
          s = fsense;
        } else {
          const double f = surf_f(k >> 1, g.surf[sid].c, rx, ry, rz);
          s = f >= 0.0;
          if (fabs(f) <= ld(g.surf_tol + sid)) nb = 1u;
        }
        ok = ok && (s == ((k & 1) ? 0 : 1));
      }
    } else {
      int szl, szh;
      {
        const int sid = rg.zsid[0];
        if (sid == fsid) szl = fsense;
        else { const double f = surf_f(S_PZ, g.surf[sid].c, rx, ry, rz); szl = f >= 0.0; if (fabs(f) <= ld(g.surf_tol + sid)) nb = 1u; }
      }
      {
        const int sid = rg.zsid[1];
        if (sid == fsid) szh = fsense;
        else { const double f = surf_f(S_PZ, g.surf[sid].c, rx, ry, rz); szh = f >= 0.0; if (fabs(f) <= ld(g.surf_tol + sid)) nb = 1u; }
      }
      ok = szl == 1 && szh == 0;
      // annulus: first k with (k == 0 or inner sense POS) and outer sense NEG
      int found = -1, prev_pos = 1;
      uint32_t nb_in = 0, nb_prev = 0;
      for (int k = 0; k < rg.n_root_cells && found < 0; ++k) {
        const int sid = rg.root_sid[k];
        int s;
        uint32_t nbk = 0;
        if (sid == fsid) s = fsense;
        else { const double f = surf_f(S_CZ, g.surf[sid].c, rx, ry, rz); s = f >= 0.0; nbk = fabs(f) <= ld(g.surf_tol + sid); }
        if (prev_pos && s == 0) { found = k; nb_in = nb_prev | nbk; }
        prev_pos = s;
        nb_prev = nbk;
      }
      ok = ok && found >= 0;
      nb |= nb_in;
      ann = found < 0 ? 0 : found;
      core = ann == 0;
      if (ok && !core) mc = rg.root_mc[ann];
    }
    st.a(0) = ann;
    if (ok) flags |= nb;
    if (ok && core) {
      const double trx = ld(g.cell_tr + 3 * rg.root_fill_cell), try_ = ld(g.cell_tr + 3 * rg.root_fill_cell + 1),
                   trz = ld(g.cell_tr + 3 * rg.root_fill_cell + 2);
      st.set_u(1, rg.root_univ_child, K > 0 ? U_RECT : U_CSG);
      st.setT(1, 0, 0.0 + trx);
      st.setT(1, 1, 0.0 + try_);
      st.setT(1, 2, 0.0 + trz);
    }
  }
  // rect levels (Alg. 5 per level; translations accumulate as in the generic descent)
#pragma unroll
  for (int lv = 1; lv <= kRectMaxK; ++lv) {
    if (lv <= K && ok && core && lv >= l0) {
      const DUniv* U = g.univ + st.u(lv);
      const double Tx = st.T(lv, 0), Ty = st.T(lv, 1), Tz = st.T(lv, 2);
      const double x = rx - Tx, y = ry - Ty, z = rz - Tz;
      const double llx = ld(&U->d[0]), lly = ld(&U->d[1]), px = ld(&U->d[3]), py = ld(&U->d[4]);
      const int i = rect_index(llx, px, x), j = rect_index(lly, py, y);
      uint32_t nb = near_wall(llx, px, i, x) | near_wall(lly, py, j, y);
      int k = 0;
      if (!ld(&U->is2d)) {
        const double llz = ld(&U->d[2]), pz = ld(&U->d[5]);
        k = rect_index(llz, pz, z);
        nb |= near_wall(llz, pz, k, z);
      }
      flags |= nb;
      st.a(lv) = i; st.b(lv) = j; st.c(lv) = k;
      double tx, ty, tz;
      const int dau = array_daughter(g, U, U_RECT, i, j, k, tx, ty, tz);
      if (dau < 0) {
        ok = false;
      } else {
        st.set_u(lv + 1, dau, lv < K ? U_RECT : U_CSG);
        st.setT(lv + 1, 0, Tx + tx);
        st.setT(lv + 1, 1, Ty + ty);
        st.setT(lv + 1, 2, Tz + tz);
      }
    }
  }
  // pin (concentric CZs): annulus = first k with (k == 0 or inner POS) and outer NEG
  if (ok && core) {
    const int pin = ld(rg.pin_of_univ + st.u(KP));
    const int off = ld(rg.pin_off + pin), ncz = ld(rg.pin_off + pin + 1) - off;
    const double x = rx - st.T(KP, 0), y = ry - st.T(KP, 1), z = rz - st.T(KP, 2);
    const int psid = l0 == KP ? fsid : -1;
    int a = ncz, prev_pos = 1;
    uint32_t nb_prev = 0, nb_in = 0;
    for (int k = 0; k < ncz; ++k) {
      const int sid = ld(rg.pin_sid + off + k);
      int s;
      uint32_t nbk = 0;
      if (sid == psid) s = fsense;
      else { const double f = surf_f(S_CZ, g.surf[sid].c, x, y, z); s = f >= 0.0; nbk = fabs(f) <= ld(g.surf_tol + sid); }
      if (prev_pos && s == 0) { a = k; nb_in = nb_prev | nbk; break; }
      prev_pos = s;
      nb_prev = nbk;
    }
    if (a == ncz) { nb_in = nb_prev; if (!prev_pos) ok = false; }
    flags |= nb_in;
    st.a(KP) = pin;
    st.b(KP) = a;
    mc = ld(rg.pin_mc + off + pin + a);
  }
  L = core ? K + 2 : 1;
  return ok;
}

// distance_to_boundary over the RTK stack, in the generic tracker's canonical order (O13)
template <bool BOX>
__device__ __forceinline__ void rect_distances(const DevGeom& g, const RectGeom& rg, Stack& st, int L, double rx,
                                               double ry, double rz, double u, double v, double w, int os_l,
                                               int os_s, Best& b) {
  const int K = rg.K, KP = K + 1;
  // level 0: the root cell's half-spaces in surface-id order
  if (BOX) {
#pragma unroll
    for (int k = 0; k < 6; ++k) {
      const int sid = rg.box_sid[k];
      const double d = surf_dist(k >> 1, (k & 1) ? 0 : 1, false, g.surf[sid].c, rx, ry, rz, u, v, w);
      b.consider(d, 0, sid, (k & 1) ? 0 : 1);
    }
  } else {
    const int ann = st.a(0);
    {
      const int sid = rg.zsid[0];
      const double d = surf_dist(S_PZ, 1, false, g.surf[sid].c, rx, ry, rz, u, v, w);
      b.consider(d, 0, sid, 1);
    }
    {
      const int sid = rg.zsid[1];
      const double d = surf_dist(S_PZ, 0, false, g.surf[sid].c, rx, ry, rz, u, v, w);
      b.consider(d, 0, sid, 0);
    }
    if (ann > 0) {
      const int sid = rg.root_sid[ann - 1];
      const double d = surf_dist(S_CZ, 1, os_l == 0 && os_s == sid, g.surf[sid].c, rx, ry, rz, u, v, w);
      b.consider(d, 0, sid, 1);
    }
    {
      const int sid = rg.root_sid[ann];
      const double d = surf_dist(S_CZ, 0, os_l == 0 && os_s == sid, g.surf[sid].c, rx, ry, rz, u, v, w);
      b.consider(d, 0, sid, 0);
    }
  }
  if (L > 1) {
#pragma unroll
    for (int lv = 1; lv <= kRectMaxK; ++lv) {
      if (lv <= K) {
        const DUniv* U = g.univ + st.u(lv);
        const double x = rx - st.T(lv, 0), y = ry - st.T(lv, 1), z = rz - st.T(lv, 2);
        const int i = st.a(lv), j = st.b(lv);
        if (u != 0.0) b.consider(rect_wall(ld(&U->d[0]), ld(&U->d[3]), i, x, u), lv, u > 0.0 ? 1 : 0, 0);
        if (v != 0.0) b.consider(rect_wall(ld(&U->d[1]), ld(&U->d[4]), j, y, v), lv, v > 0.0 ? 3 : 2, 0);
        if (!ld(&U->is2d) && w != 0.0)
          b.consider(rect_wall(ld(&U->d[2]), ld(&U->d[5]), st.c(lv), z, w), lv, w > 0.0 ? 5 : 4, 0);
      }
    }
    // pin: inner cylinder (outside of it), then outer cylinder (inside of it)
    const int pin = st.a(KP), pa = st.b(KP);
    const int off = ld(rg.pin_off + pin), ncz = ld(rg.pin_off + pin + 1) - off;
    const double x = rx - st.T(KP, 0), y = ry - st.T(KP, 1), z = rz - st.T(KP, 2);
    if (pa > 0) {
      const int sid = ld(rg.pin_sid + off + pa - 1);
      const double d = surf_dist(S_CZ, 1, os_l == KP && os_s == sid, g.surf[sid].c, x, y, z, u, v, w);
      b.consider(d, KP, sid, 1);
    }
    if (pa < ncz) {
      const int sid = ld(rg.pin_sid + off + pa);
      const double d = surf_dist(S_CZ, 0, os_l == KP && os_s == sid, g.surf[sid].c, x, y, z, u, v, w);
      b.consider(d, KP, sid, 0);
    }
  }
}

NT_DEV_END
