// Dynamic-polymorphism (DP) dispatch of the tracking operations (§4.1 "Dynamic
// polymorphism (DP) method").
//
// The paper's DP method defines the Table 1 operations as pure virtual methods of a
// tracker base class, with CSG and rectilinear-array trackers deriving from it, and a polymorphic
// get_tracker returning a pointer to the universe's tracker.  Here the same structure is built on
// the device: k_dp_init placement-constructs one tracker object per universe in device memory
// (so the vtable pointers belong to this CUDA module) and stores a pointer table; the event
// kernel instantiated with DP = true reaches find_cell, distance_to_boundary and the array
// cross_surface step only through those virtual calls (indirect CALL in SASS, no inlining).
// The SP method is the default kernel (switch on the universe kind); ST is the
// pseudo-array build option (every universe CSG).
//
// Every virtual method calls the same nt_geom.cuh arithmetic as the SP path, so DP walks are
// bit-identical to SP and to the oracle (tested).
#pragma once
#include <new>

NT_DEV_BEGIN

struct UnivTracker {
  const DUniv* U;
  // Alg. 7 step at one level: locate the cell / tile of (x, y, z) in this universe (forced sense
  // fsid/fsense applies when fsid >= 0).  Writes the stack indices and the frame translation of
  // the daughter.  Returns the daughter universe id (>= 0), -1 when LOST, or -2 - mc for a
  // material cell.
  __device__ virtual int find_cell(const DevGeom& g, double x, double y, double z, int fsid, int fsense,
                                   int& ia, int& ib, int& ic, double& tx, double& ty, double& tz,
                                   uint32_t& flags) const = 0;
  // distance_to_boundary candidates of the current cell / tile at level l (canonical order, O13)
  __device__ virtual void distance(const DevGeom& g, int ia, int ib, int ic, int l, double x, double y,
                                   double z, double u, double v, double w, int os_l, int os_s, Best& b) const = 0;
  // Alg. 6 cross_surface in an array: tile +-1 across face j, daughter universe and translation
  // (CSG universes re-run find_cell with the forced sense instead; never called for them).
  __device__ virtual int next_tile(const DevGeom& g, int j, int& ta, int& tb, int& tc, double& tx,
                                   double& ty, double& tz) const = 0;
};

struct CsgTracker final : UnivTracker {
  __device__ int find_cell(const DevGeom& g, double x, double y, double z, int fsid, int fsense, int& ia,
                           int& ib, int& ic, double& tx, double& ty, double& tz,
                           uint32_t& flags) const override {
    int f = 0;
    int h0 = 0, h1 = 0;
    const int cell = csg_find(g, ld(&U->i0), x, y, z, fsid, fsense, flags, f, h0, h1);
    if (cell < 0) return -1;
    ia = cell; ib = 0; ic = 0;
    if (f >= 0) return -2 - f;
    tx = ld(g.cell_tr + 3 * cell);
    ty = ld(g.cell_tr + 3 * cell + 1);
    tz = ld(g.cell_tr + 3 * cell + 2);
    return -1 - f;
  }
  __device__ void distance(const DevGeom& g, int ia, int, int, int l, double x, double y, double z, double u,
                           double v, double w, int os_l, int os_s, Best& b) const override {
    const int h0 = ld(g.cell_hs + ia), h1 = ld(g.cell_hs + ia + 1);
    for (int h = h0; h < h1; ++h) {
      const DHs* r = g.hsr + h;
      const int e = ld(&r->e);
      const int sid = hs_sid(e);
      const double d = surf_dist(hs_kind(e), hs_sense(e), os_l == l && os_s == sid, r->c, x, y, z, u, v, w);
      b.consider(d, l, h, hs_sense(e));
    }
  }
  __device__ int next_tile(const DevGeom&, int, int&, int&, int&, double&, double&, double&) const override {
    return -1;
  }
};

struct RectTracker final : UnivTracker {
  __device__ int find_cell(const DevGeom& g, double x, double y, double z, int, int, int& ia, int& ib, int& ic,
                           double& tx, double& ty, double& tz, uint32_t& flags) const override {
    int i, j, k;
    rect_locate(g, U, x, y, z, i, j, k, flags);
    ia = i; ib = j; ic = k;
    return array_daughter(g, U, U_RECT, i, j, k, tx, ty, tz);
  }
  __device__ void distance(const DevGeom& g, int ia, int ib, int ic, int l, double x, double y, double z,
                           double u, double v, double w, int, int, Best& b) const override {
    rect_candidates(g, U, ia, ib, ic, l, x, y, z, u, v, w, b);
  }
  __device__ int next_tile(const DevGeom& g, int j, int& ta, int& tb, int& tc, double& tx, double& ty,
                           double& tz) const override {
    const int dir = (j & 1) ? 1 : -1, ax = j >> 1;
    if (ax == 0) ta += dir; else if (ax == 1) tb += dir; else tc += dir;
    return array_daughter(g, U, U_RECT, ta, tb, tc, tx, ty, tz);
  }
};

struct HexTracker final : UnivTracker {
  __device__ int find_cell(const DevGeom& g, double x, double y, double z, int, int, int& ia, int& ib, int& ic,
                           double& tx, double& ty, double& tz, uint32_t& flags) const override {
    int q, r, k = 0;
    hex_locate(U, x, y, q, r, flags);
    if (ld(&U->i1) > 0) {
      const double zl = ld(&U->d[4]), zp = ld(&U->d[5]);
      k = rect_index(zl, zp, z);
      flags |= near_wall(zl, zp, k, z);
    }
    ia = q; ib = r; ic = k;
    return array_daughter(g, U, U_HEX, q, r, k, tx, ty, tz);
  }
  __device__ void distance(const DevGeom&, int ia, int ib, int ic, int l, double x, double y, double z, double u,
                           double v, double w, int, int, Best& b) const override {
    double t0, t1, t2, m0, m1, m2;
    hex_t(U, x, y, t0, t1, t2);
    hex_m(ia, ib, m0, m1, m2);
    const double p = ld(&U->d[2]);
    const double tk[3] = {t0, t1, t2}, mk[3] = {m0, m1, m2};
#pragma unroll 1
    for (int k = 0; k < 3; ++k) {
      const double gk = ld(&U->d[10 + 2 * k]) * u + ld(&U->d[11 + 2 * k]) * v;
      if (gk != 0.0) {
        const double bnd = gk > 0.0 ? mk[k] + 0.5 : mk[k] - 0.5;
        b.consider(clamp0(fdiv(p * bnd - tk[k], gk)), l, gk > 0.0 ? k : k + 3, 0);
      }
    }
    if (ld(&U->i1) > 0 && w != 0.0)
      b.consider(rect_wall(ld(&U->d[4]), ld(&U->d[5]), ic, z, w), l, w > 0.0 ? 7 : 6, 0);
  }
  __device__ int next_tile(const DevGeom& g, int j, int& ta, int& tb, int& tc, double& tx, double& ty,
                           double& tz) const override {
    if (j < 6) {
      ta += (j == 0 || j == 5) ? 1 : ((j == 2 || j == 3) ? -1 : 0);
      tb += (j == 1 || j == 2) ? 1 : ((j == 4 || j == 5) ? -1 : 0);
    } else {
      tc += (j == 7) ? 1 : -1;
    }
    return array_daughter(g, U, U_HEX, ta, tb, tc, tx, ty, tz);
  }
};

constexpr int kTrkBytes = 32;   // >= sizeof of every tracker (vptr + U)
static_assert(sizeof(CsgTracker) <= kTrkBytes && sizeof(RectTracker) <= kTrkBytes &&
              sizeof(HexTracker) <= kTrkBytes, "tracker object size");

// get_tracker: the polymorphic pointer of universe u
__device__ __forceinline__ const UnivTracker* get_tracker(const DevGeom& g, int u) {
  return reinterpret_cast<const UnivTracker* const*>(g.trk)[u];
}

// one tracker object per universe, constructed on the device (vtables of this module)
__global__ void k_dp_init(const DevGeom g, unsigned char* objs, const void** tab) {
  for (int u = blockIdx.x * blockDim.x + threadIdx.x; u < g.n_univ; u += gridDim.x * blockDim.x) {
    void* p = objs + (size_t)u * kTrkBytes;
    const DUniv* U = g.univ + u;
    UnivTracker* t;
    const int kind = U->kind;
    if (kind == U_CSG) t = new (p) CsgTracker();
    else if (kind == U_RECT) t = new (p) RectTracker();
    else t = new (p) HexTracker();
    t->U = U;
    tab[u] = t;
  }
}

// Alg. 7 descent through the virtual find_cell (same contract as descend())
template <bool STORE_T = true>
__device__ __forceinline__ bool descend_dp(const DevGeom& g, Stack& st, int l0, int u, double Tx, double Ty,
                                           double Tz, double rx, double ry, double rz, int fsid, int fsense,
                                           int& L, int& mc, uint32_t& flags) {
#pragma unroll 1
  for (int l = l0; l < kMaxDepth; ++l) {
    st.set_u(l, u, ld(&g.univ[u].kind));
    if (STORE_T) {
      st.setT(l, 0, Tx);
      st.setT(l, 1, Ty);
      st.setT(l, 2, Tz);
    }
    int ia = 0, ib = 0, ic = 0;
    double tx = 0.0, ty = 0.0, tz = 0.0;
    const int r = get_tracker(g, u)->find_cell(g, rx - Tx, ry - Ty, rz - Tz, l == l0 ? fsid : -1, fsense, ia,
                                               ib, ic, tx, ty, tz, flags);
    if (r == -1) return false;
    st.a(l) = ia; st.b(l) = ib; st.c(l) = ic;
    if (r <= -2) { L = l + 1; mc = -2 - r; return true; }
    Tx = Tx + tx;
    Ty = Ty + ty;
    Tz = Tz + tz;
    u = r;
  }
  return false;
}

__device__ __forceinline__ void level_distances_dp(const DevGeom& g, Stack& st, int l, double rx, double ry,
                                                   double rz, double u, double v, double w, int os_l, int os_s,
                                                   Best& b) {
  const double x = rx - st.T(l, 0), y = ry - st.T(l, 1), z = rz - st.T(l, 2);
  get_tracker(g, st.u(l))->distance(g, st.a(l), st.b(l), st.c(l), l, x, y, z, u, v, w, os_l, os_s, b);
}

NT_DEV_END
