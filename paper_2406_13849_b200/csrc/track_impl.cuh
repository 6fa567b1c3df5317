// Generic nested-geometry tracker for sm_100a (history-based persistent kernel).
//
// One thread owns one history at a time and walks it through Alg. 2:
// distance_to_surface over every level of the universe stack (Table 1), collide
// or cross, cross_surface at the top-most level holding the surface (Alg. 8,
// P:584-592) by BIH search or array index +-1 (Alg. 6), re-descend
// (Alg. 7), isotropic scatter / absorption.  When its history ends
// the thread claims the next pid from a global counter (persistent refill; warp-aggregated
// atomics), so the grid never drains while work remains (§2.3 vector of histories,
// P:424-434, re-designed as a persistent history-based kernel — DESIGN.md).
//
// The per-level universe stack lives in shared memory (one slot per thread per level,
// stride = blockDim, conflict-free).  Tallies: exits and counters are u32
// shared-memory atomics per block; track lengths go to the block's own fp64 slice in global
// memory (RED.F64 at L2: a shared-memory fp64 atomicAdd would be a CAS loop), and the slices
// and shared counters are flushed once per block at the end (flush_tallies).
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <type_traits>

#include "../../include/nestrack.h"
#include "nt_geom.cuh"
#include "nt_kernels.hpp"
#include "nt_layout.hpp"
#include "nt_math.cuh"

#ifndef NT_HS_UNROLL
#define NT_HS_UNROLL 1       // unroll of a CSG cell's half-space loop in distance_to_boundary (tuning)
#endif

NT_DEV_BEGIN
constexpr int kHsUnroll = NT_HS_UNROLL;
// slab pairs of axis planes evaluated with one division (builder kHsSlab), in the f0 feature set: the
// branch costs the hex models more than it saves (C4 −7 %; C1 +16 %, C2 +13 %, C3 +2.5 %, C5r +9.5 %)
#ifndef NT_SLABS
#define NT_SLABS (NT_FEAT == 0)
#endif
constexpr bool kSlabs = NT_SLABS != 0;




// per-thread universe stack in shared memory, level-major: [level][field][B] so that one
// level's fields sit at fixed offsets from one per-level base (conflict-free across a warp)
// The root frame is the global frame (T_0 = 0 always), so translations are stored from level 1.
struct Stack {
  int* si;      // [maxd][4][B]: u | kind << 28, a, b, c   (thread-offset already applied)
  double* sT;   // [maxd-1][3][B]: T of levels 1 .. maxd-1 (thread-offset already applied)
  int B;
  // the universe's kind travels with its id, so distance and crossing code need no universe load
  __device__ __forceinline__ int u(int l) const { return si[(4 * l + 0) * B] & 0x0FFFFFFF; }
  __device__ __forceinline__ int ukind(int l) const { return static_cast<int>(static_cast<unsigned>(si[(4 * l + 0) * B]) >> 28); }
  __device__ __forceinline__ void set_u(int l, int u, int kind) { si[(4 * l + 0) * B] = u | (kind << 28); }
  __device__ __forceinline__ int& a(int l) { return si[(4 * l + 1) * B]; }
  __device__ __forceinline__ int& b(int l) { return si[(4 * l + 2) * B]; }
  __device__ __forceinline__ int& c(int l) { return si[(4 * l + 3) * B]; }
  __device__ __forceinline__ double T(int l, int k) const { return l ? sT[(3 * (l - 1) + k) * B] : 0.0; }
  __device__ __forceinline__ void setT(int l, int k, double v) { if (l) sT[(3 * (l - 1) + k) * B] = v; }
};

// D1: instance of the material cell at the bottom of the stack (levels 0 .. L-1): the sum over the
// levels of the instances that precede the chosen child (builder: build_instance_tables).
__device__ __forceinline__ int instance_of(const DevGeom& g, Stack& st, int L) {
  int inst = 0;
#pragma unroll 1
  for (int l = 0; l < L; ++l) {
    const int u = st.u(l);
    const DUniv* U = g.univ + u;
    const int kind = st.ukind(l);
    int k;
    if (kind == U_CSG) {
      k = ld(g.cell_pos + st.a(l));
    } else if (!kHex || kind == U_RECT) {
      const int n0 = ld(&U->i0), n1 = ld(&U->i1), n2 = ld(&U->i2), is2d = ld(&U->is2d);
      const int a = st.a(l), b = st.b(l), c = st.c(l);
      const bool in = a >= 0 && a < n0 && b >= 0 && b < n1 && (is2d || (c >= 0 && c < n2));
      k = in ? a + n0 * (b + n1 * (is2d ? 0 : c)) : n0 * n1 * n2;
    } else {
      const int R = ld(&U->i0), nz = ld(&U->i1), W = 2 * R + 1;
      const int q = st.a(l), r = st.b(l), kz = st.c(l);
      const bool in = max(abs(q), max(abs(r), abs(q + r))) <= R && (nz == 0 || (kz >= 0 && kz < nz));
      k = in ? (nz > 0 ? kz : 0) * W * W + (r + R) * W + (q + R) : W * W * (nz > 0 ? nz : 1);
    }
    inst += ld(g.inst_off + ld(g.univ_inst + u) + k);
  }
  return inst;
}

// The distance winner's surface: for a CSG level the key holds the half-space index h; its surface
// id and surf_meta (BC) come from the record.  Array levels: the key is the wall / face number.
__device__ __forceinline__ int winner_surface(const DevGeom& g, bool csg, int jb, int& meta) {
  meta = 0;
  if (!csg) return jb;
  const DHs* r = g.hsr + jb;
  meta = ld(&r->meta) & 0xFF;     // surf_meta (the slab bit above it is the distance loop's)
  return hs_sid(ld(&r->e));
}

// Alg. 7 descent from level l0 in universe u with frame translation T.  fh >= 0: a CSG crossing
// out of the cell at level l0 through half-space entry fh; the crossed surface's sense is forced to
// fsense at level l0 (O9') and the cells across it (hs_nb_off[fh]) are tested first.  Returns false
// when a level has no cell (LOST).
// MIXED (with STORE_T): frames are stored only for levels whose parent is an array; a level below a
// CSG level has T_l = T_{l-1} + the parent cell's translation, recomputed by its readers (frame_mixed)
template <bool STORE_T = true, bool MIXED = false>
__device__ __forceinline__ bool descend(const DevGeom& g, Stack& st, int l0, int u, double Tx, double Ty,
                                     double Tz, double rx, double ry, double rz, int fh, int fsense,
                                     int& L, int& mc, uint32_t& flags) {
  int fsid = -1;
  const CRef* nbl = nullptr;
  int nnb = 0;
  if (fh >= 0) {
    fsid = hs_sid(ld(&g.hsr[fh].e));
    const int k0 = ld(g.hs_nb_off + fh);
    nbl = g.nb_cells + k0;
    nnb = ld(g.hs_nb_off + fh + 1) - k0;
  }
  bool parent_csg = false;           // MIXED: level l's parent is a CSG level (frame not stored)
#pragma unroll 1
  for (int l = l0; l < kMaxDepth; ++l) {
    const DUniv* U = g.univ + u;
    const int kind = ld(&U->kind);
    // a CSG crossing re-descends from its own level: that level's universe and frame are already
    // in the stack, unchanged
    if (!(l == l0 && fh >= 0)) {
      st.set_u(l, u, kind);
      if (STORE_T && !(MIXED && parent_csg)) {
        st.setT(l, 0, Tx);
        st.setT(l, 1, Ty);
        st.setT(l, 2, Tz);
      }
    }
    const double x = rx - Tx, y = ry - Ty, z = rz - Tz;
    double tx, ty, tz;
    int dau;
    if (kind == U_CSG) {
      const bool first = l == l0;
      int f = 0, h0 = 0, h1 = 0;
      const int cell = csg_find(g, ld(&U->i0), x, y, z, first ? fsid : -1, fsense, flags, f, h0, h1,
                                first ? nbl : nullptr, first ? nnb : 0);
      if (cell < 0) return false;
      st.a(l) = cell;
      st.b(l) = h0;                 // a CSG level keeps its cell's half-space range in b, c
      st.c(l) = h1;
      if (f >= 0) { L = l + 1; mc = f; return true; }
      dau = -1 - f;
      parent_csg = true;
      tx = ld(g.cell_tr + 3 * cell);
      ty = ld(g.cell_tr + 3 * cell + 1);
      tz = ld(g.cell_tr + 3 * cell + 2);
    } else if (!kHex || kind == U_RECT) {
      int i, j, k;
      rect_locate(g, U, x, y, z, i, j, k, flags);
      st.a(l) = i; st.b(l) = j; st.c(l) = k;
      dau = array_daughter(g, U, U_RECT, i, j, k, tx, ty, tz);
      parent_csg = false;
    } else {
      int q, r, k = 0;
      hex_locate(U, x, y, q, r, flags);
      if (ld(&U->i1) > 0) {
        const double zl = ld(&U->d[4]), zp = ld(&U->d[5]);
        k = rect_index(zl, zp, z);
        flags |= near_wall(zl, zp, k, z);
      }
      st.a(l) = q; st.b(l) = r; st.c(l) = k;
      dau = array_daughter(g, U, U_HEX, q, r, k, tx, ty, tz);
      parent_csg = false;
    }
    if (dau < 0) return false;
    Tx = Tx + tx;
    Ty = Ty + ty;
    Tz = Tz + tz;
    u = dau;
  }
  return false;
}

// distance candidates of level l in its local frame (canonical order, O13)
__device__ __forceinline__ void level_candidates(const DevGeom& g, const DUniv* U, int kind, int ia, int ib,
                                                 int ic, int l, double x, double y, double z, double u,
                                                 double v, double w, int os_l, int os_s, Best& b) {
  if (kind == U_CSG) {
    const int h0 = ib, h1 = ic;     // the cell's half-space range, kept in the stack by the descent
#pragma unroll kHsUnroll
    for (int h = h0; h < h1; ++h) {
      const DHs* r = g.hsr + h;
      const double2 c01 = __ldg(reinterpret_cast<const double2*>(r->c));
      const double2 c23 = __ldg(reinterpret_cast<const double2*>(r->c + 2));
      const int2 em = __ldg(reinterpret_cast<const int2*>(&r->e));
      const int e = em.x;
      if (kSlabs && (em.y & kHsSlab)) {
        // slab: entries h and h+1 are the same axis plane kind with opposite senses.  A plane of sense
        // 0 is exited only moving up the axis (den > 0), one of sense 1 only moving down, so at most
        // one of the two candidates is finite: that one, with surf_dist's arithmetic, at h's turn
        // (h and h+1 are adjacent in the canonical order, so ties resolve as before)
        const int kind = hs_kind(e);
        const double den = sel3(kind, u, v, w);
        const bool second = (den > 0.0) != (hs_sense(e) == 0);   // the entry exited along den's sign
        const double c0 = second ? ld(&r[1].c[0]) : c01.x;
        const int sp = second ? hs_sense(e) ^ 1 : hs_sense(e);
        const double d = dsel(den != 0.0, clamp0(fdiv(c0 - sel3(kind, x, y, z), den)), NT_INF);
        b.consider(d, l, second ? h + 1 : h, sp);
        ++h;
        continue;
      }
      const int sid = hs_sid(e);
      const double d = surf_dist(hs_kind(e), hs_sense(e), os_l == l && os_s == sid, c01.x, c01.y, c23.x, c23.y,
                                 x, y, z, u, v, w);
      b.consider(d, l, h, hs_sense(e));          // +inf (no hit) is a no-op; CSG key = half-space index
    }
  } else if (!kHex || kind == U_RECT) {
    rect_candidates(g, U, ia, ib, ic, l, x, y, z, u, v, w, b);
  } else {
    double t0, t1, t2, m0, m1, m2;
    hex_t(U, x, y, t0, t1, t2);
    hex_m(ia, ib, m0, m1, m2);
    const double p = ld(&U->d[2]);
    const double tk[3] = {t0, t1, t2}, mk[3] = {m0, m1, m2};
    // unrolled (the t / m arrays stay in registers) and branch-free: a family with g_k = 0 has no
    // forward face, +inf is a no-op for consider
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const double gk = ld(&U->d[10 + 2 * k]) * u + ld(&U->d[11 + 2 * k]) * v;
      const double bnd = dsel(gk > 0.0, mk[k] + 0.5, mk[k] - 0.5);
      b.consider(dsel(gk != 0.0, clamp0(fdiv(p * bnd - tk[k], gk)), NT_INF), l, gk > 0.0 ? k : k + 3, 0);
    }
    if (ld(&U->i1) > 0)
      b.consider(dsel(w != 0.0, rect_wall(ld(&U->d[4]), ld(&U->d[5]), ic, z, w), NT_INF), l, w > 0.0 ? 7 : 6, 0);
  }
}

// distance candidates of level l using the stored frame T_l
__device__ __forceinline__ void level_distances(const DevGeom& g, Stack& st, int l, double rx, double ry,
                                                double rz, double u, double v, double w, int os_l,
                                                int os_s, Best& b) {
  const double x = rx - st.T(l, 0), y = ry - st.T(l, 1), z = rz - st.T(l, 2);
  level_candidates(g, g.univ + st.u(l), st.ukind(l), st.a(l), st.b(l), st.c(l), l, x, y, z, u, v, w, os_l, os_s, b);
}

// ---- safety bound of a level: a lower bound on the Euclidean distance from the local
// point to every surface that can bound level l's current cell / tile.  Every distance candidate of
// the level is a ray distance to one of these surfaces along a (unit) direction, hence >= it.  The
// bound depends on the position only, so it stays valid (minus the path flown) across collisions.
// Plain |f|-style distances: rounding errors are covered by the relative / absolute margin of the
// skip test (kSafeRel, kSafeAbs in event_kernel.cuh).
__device__ __forceinline__ double hs_safety(int kind, double c0, double c1, double c2, double c3, double x, double y,
                                            double z) {
  if (kind <= S_PZ) return fabs(sel3(kind, x, y, z) - c0);
  if (kPlane && kind == S_PLANE) return fdiv(fabs(((c0 * x + c1 * y) + c2 * z) - c3), fsqrt((c0 * c0 + c1 * c1) + c2 * c2));
  const double dx = x - c0, dy = y - c1;
  if (!kSphere || kind == S_CZ) return fabs(fsqrt(dx * dx + dy * dy) - c3);        // CZ: c3 = R (builder)
  const double dz = z - c2;
  return fabs(fsqrt((dx * dx + dy * dy) + dz * dz) - fsqrt(c3));
}

// safety bound of level l in its local frame (the level's cell / tile as kept in the stack)
__device__ __forceinline__ double level_safety(const DevGeom& g, const DUniv* U, int kind, int ia, int ib, int ic,
                                               double x, double y, double z) {
  double s = NT_INF;
  if (kind == U_CSG) {
#pragma unroll 1
    for (int h = ib; h < ic; ++h) {
      const DHs* r = g.hsr + h;
      const double2 c01 = __ldg(reinterpret_cast<const double2*>(r->c));
      const double2 c23 = __ldg(reinterpret_cast<const double2*>(r->c + 2));
      s = fmin(s, hs_safety(hs_kind(ld(&r->e)), c01.x, c01.y, c23.x, c23.y, x, y, z));
    }
  } else if (!kHex || kind == U_RECT) {
    if (kRectNU && ld(&U->ntile) >= 0) {
      const int n0 = ld(&U->i0), n1 = ld(&U->i1);
      const double* ex = g.edges + ld(&U->ntile);
      const double* ey = ex + n0 + 1;
      auto nu = [&](const double* e, int n, int i, double p) {
        const double lo = i >= 0 ? p - ld(e + i) : NT_INF, hi = i + 1 <= n ? ld(e + i + 1) - p : NT_INF;
        return fmin(lo, hi);
      };
      s = fmin(nu(ex, n0, ia, x), nu(ey, n1, ib, y));
      if (!ld(&U->is2d)) s = fmin(s, nu(ey + n1 + 1, ld(&U->i2), ic, z));
    } else {
      const double llx = ld(&U->d[0]), lly = ld(&U->d[1]), px = ld(&U->d[3]), py = ld(&U->d[4]);
      s = fmin(fmin(x - (llx + static_cast<double>(ia) * px), (llx + static_cast<double>(ia + 1) * px) - x),
               fmin(y - (lly + static_cast<double>(ib) * py), (lly + static_cast<double>(ib + 1) * py) - y));
      if (!ld(&U->is2d)) {
        const double llz = ld(&U->d[2]), pz = ld(&U->d[5]);
        s = fmin(s, fmin(z - (llz + static_cast<double>(ic) * pz), (llz + static_cast<double>(ic + 1) * pz) - z));
      }
    }
  } else {
    // hex faces: n_k . (x - C) = p (m_k +- 1/2) with unit n_k (builder), then the z walls
    double t0, t1, t2, m0, m1, m2;
    hex_t(U, x, y, t0, t1, t2);
    hex_m(ia, ib, m0, m1, m2);
    const double p = ld(&U->d[2]);
    s = fmin(fmin(t0 - p * (m0 - 0.5), p * (m0 + 0.5) - t0),
             fmin(fmin(t1 - p * (m1 - 0.5), p * (m1 + 0.5) - t1), fmin(t2 - p * (m2 - 0.5), p * (m2 + 0.5) - t2)));
    if (ld(&U->i1) > 0) {
      const double llz = ld(&U->d[4]), pz = ld(&U->d[5]);
      s = fmin(s, fmin(z - (llz + static_cast<double>(ic) * pz), (llz + static_cast<double>(ic + 1) * pz) - z));
    }
  }
  return s;
}

// safety bound of the levels [0, lk) of the stack at the global point r
__device__ __forceinline__ double upper_safety(const DevGeom& g, Stack& st, int lk, double rx, double ry, double rz) {
  double s = NT_INF;
#pragma unroll 1
  for (int l = 0; l < lk; ++l)
    s = fmin(s, level_safety(g, g.univ + st.u(l), st.ukind(l), st.a(l), st.b(l), st.c(l), rx - st.T(l, 0),
                             ry - st.T(l, 1), rz - st.T(l, 2)));
  return s;
}

// translation from the frame of level l to the frame of level l+1 (same arithmetic as descend)
__device__ __forceinline__ void level_translation(const DevGeom& g, const DUniv* U, int kind, int ia, int ib,
                                                  int ic, double& tx, double& ty, double& tz) {
  if (kind == U_CSG) {
    tx = ld(g.cell_tr + 3 * ia);
    ty = ld(g.cell_tr + 3 * ia + 1);
    tz = ld(g.cell_tr + 3 * ia + 2);
  } else {
    array_centre(g, U, kind, ia, ib, ic, tx, ty, tz);
  }
}

// frame T_l under the MIXED policy: the nearest stored frame at or above l (or T_0 = 0), plus the
// translations of the CSG cells below it, added in level order as the descent did
__device__ __forceinline__ void frame_mixed(const DevGeom& g, Stack& st, int l, double& Tx, double& Ty, double& Tz) {
  int k = l;
  while (k > 0 && st.ukind(k - 1) == U_CSG) --k;       // level k's frame is stored (or k == 0)
  Tx = st.T(k, 0); Ty = st.T(k, 1); Tz = st.T(k, 2);
#pragma unroll 1
  for (int m = k; m < l; ++m) {
    const int c = st.a(m);
    Tx = Tx + ld(g.cell_tr + 3 * c); Ty = Ty + ld(g.cell_tr + 3 * c + 1); Tz = Tz + ld(g.cell_tr + 3 * c + 2);
  }
}

// frame T_l of level l of the stack, accumulated from level 0 (T_0 = 0) with the descent's arithmetic
__device__ __forceinline__ void frame_of(const DevGeom& g, Stack& st, int l, double& Tx, double& Ty, double& Tz) {
  Tx = 0.0; Ty = 0.0; Tz = 0.0;
#pragma unroll 1
  for (int k = 0; k < l; ++k) {
    double tx, ty, tz;
    level_translation(g, g.univ + st.u(k), st.ukind(k), st.a(k), st.b(k), st.c(k), tx, ty, tz);
    Tx = Tx + tx; Ty = Ty + ty; Tz = Tz + tz;
  }
}

template <bool TRACE>
__device__ __forceinline__ void emit(const KRun& R, uint64_t pid, uint32_t seg, int kind, int level, int j,
                                     int cb, int ca, double s, int terminal, uint32_t flags) {
  if (!TRACE) return;
  const unsigned long long slot = atomicAdd(R.trace_count, 1ull);
  if (slot >= R.trace_cap) return;
  nt_trace_rec t;
  t.pid = pid; t.s = s; t.seg = seg; t.cell_before = cb; t.cell_after = ca; t.j = j;
  t.kind = (uint8_t)kind; t.level = (int8_t)level; t.terminal = (uint8_t)terminal; t.pad = 0;
  t.flags = flags;
  R.trace[slot] = t;
}

// block tallies -> caller's packed output; the per-block length slice is re-zeroed for reuse
__device__ __forceinline__ void flush_tallies(const KRun& R, double* gl, const unsigned int* s_exit,
                                              const unsigned int* s_cnt, int nmc, int tid, int B) {
  for (int i = tid; i < nmc; i += B) {
    const double len = gl[i];
    if (len != 0.0) { atomicAdd(R.out + i, len); gl[i] = 0.0; }
    if (s_exit[i]) atomicAdd(R.out + nmc + i, static_cast<double>(s_exit[i]));
  }
  for (int i = tid; i < kNC; i += B)
    if (s_cnt[i]) atomicAdd(R.out + 2 * nmc + i, static_cast<double>(s_cnt[i]));
}

enum { C_PART = 0, C_SEG, C_CROSS, C_REFL, C_LEAK, C_COLL, C_ABS, C_LOST, C_CAP, C_FLAG, C_CBL0 };

template <bool TRACE, bool STATES, int TALLY = 0>
__global__ void __launch_bounds__(256, 3) k_track_generic(const DevGeom g, const KRun R) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int B = blockDim.x, tid = threadIdx.x, lane = tid & 31;
  const int nmc = g.n_mc;
  double* sT = reinterpret_cast<double*>(smem);
  unsigned int* s_cnt = reinterpret_cast<unsigned int*>(sT + 3 * (g.max_depth - 1) * B + 4 * g.max_depth * B / 2);
  unsigned int* s_exit = s_cnt + kNC;
  double* gl = R.slices + (size_t)blockIdx.x * nmc;   // per-block track-length tally (global)
  Stack st;
  st.sT = sT + tid;
  st.si = reinterpret_cast<int*>(sT + 3 * (g.max_depth - 1) * B) + tid;
  st.B = B;
  for (int i = tid; i < nmc; i += B) s_exit[i] = 0u;
  for (int i = tid; i < kNC; i += B) s_cnt[i] = 0u;
  __syncthreads();

  // particle state (registers)
  double rx = 0, ry = 0, rz = 0, u = 0, v = 0, w = 0, tau = 0;
  uint64_t pid = 0, idx = 0;
  uint32_t epoch = 0, flags = 0, nseg = 0, ncross = 0, ncoll = 0;
  int L = 0, mc = 0, os_l = -1, os_s = -1;
  // phase: 0 = needs a history, 1 = needs a descent, 2 = moving
  int phase = 0;
  // pending descent
  int d_l0 = 0, d_u = 0, d_fh = -1, d_fsense = 0;
  double d_Tx = 0, d_Ty = 0, d_Tz = 0;
  // pending crossing record (trace only)
  int p_l = -1, p_j = -1, p_cb = -1;
  double p_s = 0;
  const uint32_t max_seg = static_cast<uint32_t>(R.max_seg);

  for (;;) {
    int term = NT_T_NONE;
    if (phase == 0) {
      // ---- claim the next history (warp-aggregated atomic) and give birth (W1, O17-O18)
      const unsigned mask = __activemask();
      const int leader = __ffs(mask) - 1;
      const int rank = __popc(mask & ((1u << lane) - 1u));
      unsigned long long base = 0;
      if (lane == leader) base = atomicAdd(R.counter, static_cast<unsigned long long>(__popc(mask)));
      base = __shfl_sync(mask, base, leader);
      idx = base + rank;
      if (idx >= R.n) break;
      pid = R.pid0 + idx;
      double xa, xb;
      draw2(R.seed, pid, 0, 0, xa, xb);
      const double xi_tau = xb;
      if (STATES) {
        rx = R.states[idx]; ry = R.states[R.n + idx]; rz = R.states[2 * R.n + idx];
        u = R.states[3 * R.n + idx]; v = R.states[4 * R.n + idx]; w = R.states[5 * R.n + idx];
      } else {
        double xmu, xphi, xx, xy, xz, unused;
        draw2(R.seed, pid, 0, 1, xmu, xphi);
        draw2(R.seed, pid, 0, 2, xx, xy);
        draw2(R.seed, pid, 0, 3, xz, unused);
        rx = R.lo[0] + R.w[0] * xx;
        ry = R.lo[1] + R.w[1] * xy;
        rz = R.lo[2] + R.w[2] * xz;
        isotropic(xmu, xphi, u, v, w);
      }
      tau = -spec_log(xi_tau);
      epoch = 0; flags = 0; nseg = 0; ncross = 0; ncoll = 0; os_l = -1; os_s = -1;
      d_l0 = 0; d_u = g.root; d_Tx = d_Ty = d_Tz = 0.0; d_fh = -1; d_fsense = 0;
      p_l = -2;   // no pending crossing record: a failure here is a birth loss
      phase = 1;
    }
    if (phase == 1) {
      // ---- Alg. 7 / Alg. 8 descent (single call site for birth and every crossing)
      const bool ok = descend(g, st, d_l0, d_u, d_Tx, d_Ty, d_Tz, rx, ry, rz, d_fh, d_fsense, L, mc, flags);
      if (!ok) {
        flags |= NT_F3;
        term = NT_T_LOST;
        if (p_l == -2) emit<TRACE>(R, pid, 0, NT_EV_CROSS, -1, -1, -1, -1, 0.0, NT_T_LOST, flags);
        else emit<TRACE>(R, pid, nseg - 1, NT_EV_CROSS, p_l, p_j, p_cb, -1, p_s, NT_T_LOST, flags);
      } else {
        if (p_l != -2)
          emit<TRACE>(R, pid, nseg - 1, NT_EV_CROSS, p_l, p_j, p_cb, TRACE ? ld(g.mc_cell + mc) : 0, p_s,
                      NT_T_NONE, flags);
        phase = 2;
      }
    }
    if (phase == 2) {
      // ---- one segment (W2)
      if (nseg >= max_seg) {
        flags |= NT_F3;
        term = NT_T_CAPPED;
        emit<TRACE>(R, pid, nseg, NT_EV_COLLIDE, -1, -1, ld(g.mc_cell + mc), -1, 0.0, NT_T_CAPPED, flags);
      } else {
        Best b;
        b.init();
        for (int l = 0; l < L; ++l) level_distances(g, st, l, rx, ry, rz, u, v, w, os_l, os_s, b);
        const double sig = ld(g.mc_st + mc);
        const double ds = b.d;
        const double dc = sig > 0.0 ? fdiv(tau, sig) : NT_INF;
        const double g2 = b.d2 - ds, gc = fabs(dc - ds);
        if ((g2 > 0.0 && g2 <= kFlagDist) || (gc > 0.0 && gc <= kFlagDist)) flags |= NT_F2;
        const int cell_before = TRACE ? ld(g.mc_cell + mc) : 0;
        if (ds == NT_INF && dc == NT_INF) {
          flags |= NT_F3;
          term = NT_T_LOST;
          emit<TRACE>(R, pid, nseg, NT_EV_CROSS, -1, -1, cell_before, -1, 0.0, NT_T_LOST, flags);
        } else if (ds < dc) {
          // Alg. 2 "while d < tau/Sigma": tau -= Sigma d, move, cross
          const double s = ds;
          atomicAdd(gl + mc, s);
          if (TALLY & 1) mesh_score(g, R.mesh, rx, ry, rz, u, v, w, s);
          if (TALLY & 2) atomicAdd(R.inst + instance_of(g, st, L), s);
          rx = rx + s * u; ry = ry + s * v; rz = rz + s * w;
          const double tt = tau - sig * s;
          tau = tt > 0.0 ? tt : 0.0;
          ++nseg;
          const int l = b.l(), jb = b.j();
          const int kind_l = st.ukind(l);
          int meta;
          const int j = winner_surface(g, kind_l == U_CSG, jb, meta);
          const int bc = l == 0 ? meta >> 4 : 0;
          if (bc == NT_BC_VACUUM) {
            atomicAdd(s_exit + mc, 1u);
            ++ncross;
            term = NT_T_LEAKED;
            emit<TRACE>(R, pid, nseg - 1, NT_EV_LEAK, 0, j, cell_before, -1, s, NT_T_LEAKED, flags);
          } else if (bc == NT_BC_REFLECT) {
            const int ax = meta & 15;
            if (ax == 0) u = -u; else if (ax == 1) v = -v; else w = -w;
            os_l = 0; os_s = j;
            emit<TRACE>(R, pid, nseg - 1, NT_EV_REFLECT, 0, j, cell_before, cell_before, s, NT_T_NONE, flags);
          } else {
            atomicAdd(s_exit + mc, 1u);
            ++ncross;
            atomicAdd(s_cnt + C_CBL0 + l, 1u);
            const int ul = st.u(l);
            const DUniv* U = g.univ + ul;
            const int kind = kind_l;
            p_l = l; p_j = j; p_cb = cell_before; p_s = s;
            if (kind == U_CSG) {   // O9': far side of surface j in universe(l)
              d_l0 = l; d_u = ul; d_Tx = st.T(l, 0); d_Ty = st.T(l, 1); d_Tz = st.T(l, 2);
              d_fh = jb; d_fsense = b.sense() ^ 1;
              os_l = l; os_s = j;
              phase = 1;
            } else {               // Alg. 6: tile +- 1, then the new tile's daughter
              int ta = st.a(l), tb = st.b(l), tc = st.c(l);
              if (!kHex || kind == U_RECT) {
                const int dir = (j & 1) ? 1 : -1, ax = j >> 1;
                if (ax == 0) ta += dir; else if (ax == 1) tb += dir; else tc += dir;
              } else if (j < 6) {
                ta += (j == 0 || j == 5) ? 1 : ((j == 2 || j == 3) ? -1 : 0);
                tb += (j == 1 || j == 2) ? 1 : ((j == 4 || j == 5) ? -1 : 0);
              } else {
                tc += (j == 7) ? 1 : -1;
              }
              st.a(l) = ta; st.b(l) = tb; st.c(l) = tc;
              double tx, ty, tz;
              const int dau = array_daughter(g, U, kind, ta, tb, tc, tx, ty, tz);
              os_l = -1; os_s = -1;
              if (dau < 0) {
                flags |= NT_F3;
                term = NT_T_LOST;
                emit<TRACE>(R, pid, nseg - 1, NT_EV_CROSS, l, j, cell_before, -1, s, NT_T_LOST, flags);
              } else {
                d_l0 = l + 1; d_u = dau;
                d_Tx = st.T(l, 0) + tx; d_Ty = st.T(l, 1) + ty; d_Tz = st.T(l, 2) + tz;
                d_fh = -1; d_fsense = 0;
                phase = 1;
              }
            }
          }
        } else {
          // ---- collision at tau / Sigma_t: absorb or scatter isotropically (O14, O15)
          const double s = dc;
          atomicAdd(gl + mc, s);
          if (TALLY & 1) mesh_score(g, R.mesh, rx, ry, rz, u, v, w, s);
          if (TALLY & 2) atomicAdd(R.inst + instance_of(g, st, L), s);
          rx = rx + s * u; ry = ry + s * v; rz = rz + s * w;
          ++nseg;
          ++ncoll;
          os_l = -1; os_s = -1;
          ++epoch;
          double xa, xb;
          draw2(R.seed, pid, epoch, 0, xa, xb);
          if (xa < ld(g.mc_pabs + mc)) {
            term = NT_T_ABSORBED;
            if (R.bank) bank_sites(g, R.bank, R.bank_n, mc, idx, xb, rx, ry, rz);
            emit<TRACE>(R, pid, nseg - 1, NT_EV_COLLIDE, -1, -1, cell_before, cell_before, s, NT_T_ABSORBED,
                        flags);
          } else {
            double xmu, xphi;
            draw2(R.seed, pid, epoch, 1, xmu, xphi);
            isotropic(xmu, xphi, u, v, w);
            tau = -spec_log(xb);
            emit<TRACE>(R, pid, nseg - 1, NT_EV_COLLIDE, -1, -1, cell_before, cell_before, s, NT_T_NONE, flags);
          }
        }
      }
      if (term == NT_T_NONE) continue;
    }
    // ---- history ended: per-history counters into the block tallies
    phase = 0;
    atomicAdd(s_cnt + C_PART, 1u);
    atomicAdd(s_cnt + C_SEG, nseg);
    atomicAdd(s_cnt + C_CROSS, ncross);
    atomicAdd(s_cnt + C_COLL, ncoll);
    atomicAdd(s_cnt + C_REFL, nseg - ncross - ncoll);
    const int tcn = term == NT_T_ABSORBED ? C_ABS : term == NT_T_LEAKED ? C_LEAK : term == NT_T_LOST ? C_LOST : C_CAP;
    atomicAdd(s_cnt + tcn, 1u);
    if (flags) atomicAdd(s_cnt + C_FLAG, 1u);
    if (R.pflags) R.pflags[idx] = static_cast<uint8_t>(flags);
    if (R.pnseg) R.pnseg[idx] = nseg;
    if (R.pterm) R.pterm[idx] = static_cast<uint8_t>(term);
  }

  __syncthreads();
  flush_tallies(R, gl, s_exit, s_cnt, nmc, tid, B);
}

NT_DEV_END
#include "dp_tracker.cuh"
#include "rect_geom.cuh"
#include "event_kernel.cuh"
#include "wq_kernel.cuh"
#if NT_FEAT == 0
#include "rect_kernel.cuh"
#endif
NT_DEV_BEGIN

#if !defined(NT_RECT_TU) && !defined(NT_EVENT_TU)
// point location for unit parity (Alg. 7)
__global__ void __launch_bounds__(256) k_find_cells(const DevGeom g, const double* xyz, uint64_t n,
                                                    int32_t* cell_out, uint8_t* flag_out) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int B = blockDim.x;
  Stack st;
  st.sT = reinterpret_cast<double*>(smem) + threadIdx.x;
  st.si = reinterpret_cast<int*>(reinterpret_cast<double*>(smem) + 3 * (g.max_depth - 1) * B) + threadIdx.x;
  st.B = B;
  for (uint64_t i = blockIdx.x * (uint64_t)B + threadIdx.x; i < n; i += (uint64_t)gridDim.x * B) {
    int L = 0, mc = 0;
    uint32_t fl = 0;
    const bool ok = descend(g, st, 0, g.root, 0.0, 0.0, 0.0, xyz[i], xyz[n + i], xyz[2 * n + i], -1, 0, L, mc, fl);
    cell_out[i] = ok ? ld(g.mc_cell + mc) : -1;
    if (flag_out) flag_out[i] = static_cast<uint8_t>(fl | (ok ? 0u : NT_F3));
  }
}

#endif  // !NT_RECT_TU && !NT_EVENT_TU

// ---------------------------------------------------------------- host launchers
size_t generic_smem_bytes(const DevGeom& g, int block) {
  return (size_t)block * ((g.max_depth - 1) * 3 * 8 + g.max_depth * 4 * 4) + (kNC + (size_t)g.n_mc) * 4;
}

// stream-ordered scratch from the model's own memory pool (capi.cpp: nt_finalize creates it with a
// 64 MB release threshold, so synchronised launches do not re-map it), else the device default pool
template <class T>
static cudaError_t scratch_alloc(const DevGeom& g, T** p, size_t bytes, cudaStream_t stream) {
  void* v = nullptr;
  const cudaError_t e = g.pool ? cudaMallocFromPoolAsync(&v, bytes, static_cast<cudaMemPool_t>(g.pool), stream)
                               : cudaMallocAsync(&v, bytes, stream);
  *p = static_cast<T*>(v);
  return e;
}

// per-launch scratch: per-block track-length slices (stream-ordered allocation, zeroed)
template <class Launch>
static cudaError_t with_slices(const DevGeom& g, KRun R, uint64_t grid, cudaStream_t stream, Launch launch) {
  const size_t bytes = (size_t)grid * (size_t)g.n_mc * sizeof(double);
  cudaError_t e = scratch_alloc(g, &R.slices, bytes, stream);
  if (e != cudaSuccess) return e;
  e = cudaMemsetAsync(R.slices, 0, bytes, stream);
  if (e == cudaSuccess) e = launch(R);
  cudaError_t e2 = cudaFreeAsync(R.slices, stream);
  return e != cudaSuccess ? e : e2;
}

cudaError_t upload_coefficients(const double* host, int n) {
  return cudaMemcpyToSymbol(c_coef, host, sizeof(double) * n);
}

// Slots per block of the ring scheduler (block 256, SP): 320 when NT_EVENT_MINB such blocks still
// fit an SM (a warp that finishes its chunk then finds queued slots instead of waiting for the
// chunks the other seven warps hold), else 256.  NESTRACK_SLOTS=256 forces 256, any larger value the big size (tuning).
// big = 320 for the RTK kernels, kSlotsBig for the SP generic kernels (sp = true).
static int ring_slots(const DevGeom& g, bool trace, bool store_t, int nr = NQ, bool safety = false, bool sp = true) {
  static const int env = [] { const char* e = getenv("NESTRACK_SLOTS"); return e ? atoi(e) : 0; }();
  const int big = sp ? kSlotsBig : 320;
  if (env == 256) return 256;
  if (env > 256) return big;
  int dev = 0, smem_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
  const size_t need = NT_EVENT_MINB * (event_smem_bytes(g, big, trace, true, store_t, nr, safety) + 1024);
  return need <= (size_t)smem_sm ? big : 256;
}

// persistent launch of a ring / event-queue kernel: grid = SMs x occupancy (capped by the batch)
template <class Kern>
static cudaError_t launch_event_kernel(Kern kern, const DevGeom& g, const RectGeom& rg, const KRun& R, int block,
                                       size_t smem, int blocks_per_sm, cudaStream_t stream, int* grid_out) {
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int dev = 0, nsm = 0, occ = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, block, smem);
  if (e != cudaSuccess) return e;
  if (occ < 1) return cudaErrorInvalidConfiguration;
  const int bps = blocks_per_sm > 0 ? (blocks_per_sm < occ ? blocks_per_sm : occ) : occ;
  uint64_t need = (R.n + block - 1) / block, grid = (uint64_t)nsm * bps;
  if (need < grid) grid = need ? need : 1;
  *grid_out = (int)grid;
  return with_slices(g, R, grid, stream, [&](const KRun& Rs) {
    kern<<<(unsigned)grid, block, smem, stream>>>(g, Rs, rg);
    return cudaGetLastError();
  });
}

#ifdef NT_EVENT_TU
// Feature set fh (track_fh.cu: hex arrays and general planes, no spheres or non-uniform rect
// arrays): only the default path, the SP ring kernel without trace or tallies, so that its code is
// ~15 % smaller than f7's (the f7 kernel stalls on instruction fetch: profiles/r02_ncu_analysis.md).
// Everything else about such a model runs in f7.
cudaError_t launch_event_sp(const DevGeom& g, const KRun& R, bool states, int blocks_per_sm, cudaStream_t stream,
                            int* grid_out) {
  if (g.trk || R.mesh || R.inst) return cudaErrorNotSupported;
  const bool st_t = !kFramesRecompute;
  const RectGeom no_rg{};
  constexpr int SB = kSlotsBig;
  auto go = [&](auto kern, int s, int threads) -> cudaError_t {
    return launch_event_kernel(kern, g, no_rg, R, threads, event_smem_bytes(g, s, false, true, st_t, 7), blocks_per_sm,
                               stream, grid_out);
  };
  constexpr int T = kRingThreads;
  if (ring_slots(g, false, st_t, 7) == SB)
    return states ? go(k_track_event<T, false, true, false, 0, true, SB, 0, 7>, SB, T)
                  : go(k_track_event<T, false, false, false, 0, true, SB, 0, 7>, SB, T);
  return states ? go(k_track_event<256, false, true, false, 0, true, 256, 0, 7>, 256, 256)
                : go(k_track_event<256, false, false, false, 0, true, 256, 0, 7>, 256, 256);
}
#elif defined(NT_RECT_TU)
// Rect-specialised tracker (Alg. 9-10) under the ring scheduler: the same k_track_event as the
// generic tracker, with the RTK's find_cell / distance code (rect_geom.cuh).  320 slots per block
// when three blocks fit an SM (depth <= 4), else 256; trace and mesh runs use 256.
cudaError_t launch_rect_event(const DevGeom& g, const RectGeom& rg, const KRun& R, bool trace, bool states,
                              int blocks_per_sm, cudaStream_t stream, int* grid_out) {
  if (R.inst) return cudaErrorNotSupported;
  const bool mesh = R.mesh != nullptr;
  if (mesh && trace) return cudaErrorNotSupported;
  const bool s320 = !trace && !mesh && ring_slots(g, false, true, NQ, false, false) == 320;
  const size_t smem = event_smem_bytes(g, s320 ? 320 : 256, trace, true);
  auto go = [&](auto kern) {
    return launch_event_kernel(kern, g, rg, R, 256, smem, blocks_per_sm, stream, grid_out);
  };
  auto pick = [&](auto box) -> cudaError_t {
    constexpr int RT = decltype(box)::value ? 1 : 2;
    if (mesh) return states ? go(k_track_event<256, false, true, false, 1, true, 256, RT>)
                            : go(k_track_event<256, false, false, false, 1, true, 256, RT>);
    if (trace) return states ? go(k_track_event<256, true, true, false, 0, true, 256, RT>)
                             : go(k_track_event<256, true, false, false, 0, true, 256, RT>);
    if (s320) return states ? go(k_track_event<256, false, true, false, 0, true, 320, RT>)
                            : go(k_track_event<256, false, false, false, 0, true, 320, RT>);
    return states ? go(k_track_event<256, false, true, false, 0, true, 256, RT>)
                  : go(k_track_event<256, false, false, false, 0, true, 256, RT>);
  };
  return rg.root_box ? pick(std::true_type{}) : pick(std::false_type{});
}
#else

cudaError_t launch_generic(const DevGeom& g, const KRun& R, bool trace, bool states, int block,
                           int blocks_per_sm, cudaStream_t stream, int* grid_out) {
  const size_t smem = generic_smem_bytes(g, block);
  auto pick = [&](auto kern) -> cudaError_t {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int dev = 0, nsm = 0, occ = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, block, smem);
    if (e != cudaSuccess) return e;
    if (occ < 1) return cudaErrorInvalidConfiguration;
    int bps = blocks_per_sm > 0 ? (blocks_per_sm < occ ? blocks_per_sm : occ) : occ;
    uint64_t need = (R.n + block - 1) / block;
    uint64_t grid = (uint64_t)nsm * bps;
    if (need < grid) grid = need ? need : 1;
    *grid_out = (int)grid;
    return with_slices(g, R, grid, stream, [&](const KRun& Rs) {
      kern<<<(unsigned)grid, block, smem, stream>>>(g, Rs);
      return cudaGetLastError();
    });
  };
  const int tally = (R.mesh ? 1 : 0) | (R.inst ? 2 : 0);
  if (tally) {                        // tallies: separate instantiations (no extra code in the others)
    if (trace) return cudaErrorNotSupported;
    if (tally == 1) return states ? pick(k_track_generic<false, true, 1>) : pick(k_track_generic<false, false, 1>);
    if (tally == 2) return states ? pick(k_track_generic<false, true, 2>) : pick(k_track_generic<false, false, 2>);
    return states ? pick(k_track_generic<false, true, 3>) : pick(k_track_generic<false, false, 3>);
  }
  if (trace) return states ? pick(k_track_generic<true, true>) : pick(k_track_generic<true, false>);
  return states ? pick(k_track_generic<false, true>) : pick(k_track_generic<false, false>);
}

#if NT_FEAT == 0
cudaError_t launch_rect(const DevGeom& g, const RectGeom& rg, const KRun& R, bool trace, bool states,
                        int block, int blocks_per_sm, cudaStream_t stream, int* grid_out) {
  const size_t smem = (kNC + (size_t)g.n_mc) * 4;
  auto go = [&](auto kern) -> cudaError_t {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int dev = 0, nsm = 0, occ = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, block, smem);
    if (e != cudaSuccess) return e;
    if (occ < 1) return cudaErrorInvalidConfiguration;
    const int bps = blocks_per_sm > 0 ? (blocks_per_sm < occ ? blocks_per_sm : occ) : occ;
    uint64_t need = (R.n + block - 1) / block, grid = (uint64_t)nsm * bps;
    if (need < grid) grid = need ? need : 1;
    *grid_out = (int)grid;
    return with_slices(g, R, grid, stream, [&](const KRun& Rs) {
      kern<<<(unsigned)grid, block, smem, stream>>>(g, rg, Rs);
      return cudaGetLastError();
    });
  };
  auto pick_k = [&](auto box, auto tr, auto st, auto me) -> cudaError_t {
    constexpr bool BOX = decltype(box)::value, TR = decltype(tr)::value, ST = decltype(st)::value;
    constexpr int ME = decltype(me)::value ? 1 : 0;
    switch (rg.K) {
      case 0: return go(k_track_rect<0, BOX, TR, ST, ME>);
      case 1: return go(k_track_rect<1, BOX, TR, ST, ME>);
      case 2: return go(k_track_rect<2, BOX, TR, ST, ME>);
      case 3: return go(k_track_rect<3, BOX, TR, ST, ME>);
      case 4: return go(k_track_rect<4, BOX, TR, ST, ME>);
      default: return cudaErrorNotSupported;
    }
  };
  using T = std::true_type;
  using F = std::false_type;
  if (R.inst) return cudaErrorNotSupported;   // instance tallies: generic tracker only
  if (R.mesh) {                       // mesh tally: separate instantiations, no trace
    if (trace) return cudaErrorNotSupported;
    if (rg.root_box) return states ? pick_k(T{}, F{}, T{}, T{}) : pick_k(T{}, F{}, F{}, T{});
    return states ? pick_k(F{}, F{}, T{}, T{}) : pick_k(F{}, F{}, F{}, T{});
  }
  if (rg.root_box) {
    if (trace) return states ? pick_k(T{}, T{}, T{}, F{}) : pick_k(T{}, T{}, F{}, F{});
    return states ? pick_k(T{}, F{}, T{}, F{}) : pick_k(T{}, F{}, F{}, F{});
  }
  if (trace) return states ? pick_k(F{}, T{}, T{}, F{}) : pick_k(F{}, T{}, F{}, F{});
  return states ? pick_k(F{}, F{}, T{}, F{}) : pick_k(F{}, F{}, F{}, F{});
}

#else
cudaError_t launch_rect(const DevGeom&, const RectGeom&, const KRun&, bool, bool, int, int, cudaStream_t, int*) {
  return cudaErrorNotSupported;   // rect-specialisable models always use feature set 0
}
#endif

cudaError_t launch_event(const DevGeom& g, const KRun& R, bool trace, bool states, int block,
                         int blocks_per_sm, cudaStream_t stream, int* grid_out, bool async) {
  const bool st_t = g.trk != nullptr || !kFramesRecompute;     // DP kernels keep frames in smem
  size_t smem = event_smem_bytes(g, block, trace, async, st_t);
  const RectGeom no_rg{};
  auto go = [&](auto kern) -> cudaError_t {
    return launch_event_kernel(kern, g, no_rg, R, block, smem, blocks_per_sm, stream, grid_out);
  };
  const int tally = (R.mesh ? 1 : 0) | (R.inst ? 2 : 0);
  if (tally && trace) return cudaErrorNotSupported;
  if (async && block == 192) {     // ring queues, 6 warps per block (more blocks per SM)
    if (g.trk || tally) return cudaErrorNotSupported;
    smem = event_smem_bytes(g, block, trace, async, st_t, NQ, kSafeSP);
    if (trace) return states ? go(k_track_event<192, true, true, false, 0, true>) : go(k_track_event<192, true, false, false, 0, true>);
    return states ? go(k_track_event<192, false, true, false, 0, true>) : go(k_track_event<192, false, false, false, 0, true>);
  }
  if (async) {                     // barrier-free ring queues (block 256), SP or DP dispatch
    if (block != 256) return cudaErrorInvalidValue;
    constexpr int SB = kSlotsBig;
    auto pick = [&](auto dp) -> cudaError_t {
      constexpr bool D = decltype(dp)::value;
      const bool sf = !D && kSafeSP;   // SP kernels carry the safety skip's per-slot state and U ring
      smem = event_smem_bytes(g, 256, trace, true, st_t, NQ, sf);
      if (!D && tally && ring_slots(g, false, st_t, NQ, sf) == SB) {   // mesh / instance tallies: big slots as well
        smem = event_smem_bytes(g, SB, false, true, st_t, NQ, sf);
        if (tally == 1) return states ? go(k_track_event<256, false, true, false, 1, true, SB>) : go(k_track_event<256, false, false, false, 1, true, SB>);
        if (tally == 2) return states ? go(k_track_event<256, false, true, false, 2, true, SB>) : go(k_track_event<256, false, false, false, 2, true, SB>);
        return states ? go(k_track_event<256, false, true, false, 3, true, SB>) : go(k_track_event<256, false, false, false, 3, true, SB>);
      }
      if (tally == 1) return states ? go(k_track_event<256, false, true, D, 1, true>) : go(k_track_event<256, false, false, D, 1, true>);
      if (tally == 2) return states ? go(k_track_event<256, false, true, D, 2, true>) : go(k_track_event<256, false, false, D, 2, true>);
      if (tally == 3) return states ? go(k_track_event<256, false, true, D, 3, true>) : go(k_track_event<256, false, false, D, 3, true>);
#if (NT_FEAT != 0 || NT_DEPTH_RINGS_F0) && NT_DEPTH_RINGS
      if (!D) {                    // hex / plane / sphere models: depth-class rings (NR = 7)
        if (ring_slots(g, trace, st_t, 7, sf) == SB) {
          smem = event_smem_bytes(g, SB, trace, true, st_t, 7, sf);
          if (trace) return states ? go(k_track_event<256, true, true, false, 0, true, SB, 0, 7>) : go(k_track_event<256, true, false, false, 0, true, SB, 0, 7>);
          return states ? go(k_track_event<256, false, true, false, 0, true, SB, 0, 7>) : go(k_track_event<256, false, false, false, 0, true, SB, 0, 7>);
        }
        smem = event_smem_bytes(g, 256, trace, true, st_t, 7, sf);
        if (trace) return states ? go(k_track_event<256, true, true, false, 0, true, 256, 0, 7>) : go(k_track_event<256, true, false, false, 0, true, 256, 0, 7>);
        return states ? go(k_track_event<256, false, true, false, 0, true, 256, 0, 7>) : go(k_track_event<256, false, false, false, 0, true, 256, 0, 7>);
      }
#endif
      if (!D && ring_slots(g, trace, st_t, NQ, sf) == SB) {
        smem = event_smem_bytes(g, SB, trace, true, st_t, NQ, sf);
        if (trace) return states ? go(k_track_event<256, true, true, false, 0, true, SB>) : go(k_track_event<256, true, false, false, 0, true, SB>);
        if constexpr (kRingThreads != 256) {
          auto gt = [&](auto kern) -> cudaError_t {
            return launch_event_kernel(kern, g, no_rg, R, kRingThreads, smem, blocks_per_sm, stream, grid_out);
          };
          return states ? gt(k_track_event<kRingThreads, false, true, false, 0, true, SB>)
                        : gt(k_track_event<kRingThreads, false, false, false, 0, true, SB>);
        }
        return states ? go(k_track_event<256, false, true, false, 0, true, SB>) : go(k_track_event<256, false, false, false, 0, true, SB>);
      }
      if (!D && !trace && !sf) {   // deep models: two 320-thread blocks of 400 slots per SM, if they fit
        int dev = 0, smem_sm = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
        const size_t sd = event_smem_bytes(g, kDeepSlots, false, true, st_t, NQ);
        if (2 * (sd + 1024) <= (size_t)smem_sm) {
          smem = sd;
          auto gd = [&](auto kern) -> cudaError_t {
            return launch_event_kernel(kern, g, no_rg, R, kDeepThreads, smem, blocks_per_sm, stream, grid_out);
          };
          return states ? gd(k_track_event<kDeepThreads, false, true, false, 0, true, kDeepSlots>)
                        : gd(k_track_event<kDeepThreads, false, false, false, 0, true, kDeepSlots>);
        }
      }
      if (trace) return states ? go(k_track_event<256, true, true, D, 0, true>) : go(k_track_event<256, true, false, D, 0, true>);
      return states ? go(k_track_event<256, false, true, D, 0, true>) : go(k_track_event<256, false, false, D, 0, true>);
    };
    return g.trk ? pick(std::true_type{}) : pick(std::false_type{});
  }
  if (g.trk) {                     // DP dispatch (virtual tracker calls), block 256 only
    if (block != 256) return cudaErrorInvalidValue;
    if (tally == 1) return states ? go(k_track_event<256, false, true, true, 1>) : go(k_track_event<256, false, false, true, 1>);
    if (tally) return cudaErrorNotSupported;     // DP with instance tallies: ring scheduler only
    if (trace) return states ? go(k_track_event<256, true, true, true>) : go(k_track_event<256, true, false, true>);
    return states ? go(k_track_event<256, false, true, true>) : go(k_track_event<256, false, false, true>);
  }
  if (tally) {                     // tallies: separate instantiations (no extra code in the others)
    if (block == 128) {
      if (tally == 1) return states ? go(k_track_event<128, false, true, false, 1>) : go(k_track_event<128, false, false, false, 1>);
      if (tally == 2) return states ? go(k_track_event<128, false, true, false, 2>) : go(k_track_event<128, false, false, false, 2>);
      return states ? go(k_track_event<128, false, true, false, 3>) : go(k_track_event<128, false, false, false, 3>);
    }
    if (block != 256) return cudaErrorInvalidValue;
    if (tally == 1) return states ? go(k_track_event<256, false, true, false, 1>) : go(k_track_event<256, false, false, false, 1>);
    if (tally == 2) return states ? go(k_track_event<256, false, true, false, 2>) : go(k_track_event<256, false, false, false, 2>);
    return states ? go(k_track_event<256, false, true, false, 3>) : go(k_track_event<256, false, false, false, 3>);
  }
  if (block == 128) {
    if (trace) return states ? go(k_track_event<128, true, true>) : go(k_track_event<128, true, false>);
    return states ? go(k_track_event<128, false, true>) : go(k_track_event<128, false, false>);
  }
  if (block != 256) return cudaErrorInvalidValue;
  if (trace) return states ? go(k_track_event<256, true, true>) : go(k_track_event<256, true, false>);
  return states ? go(k_track_event<256, false, true>) : go(k_track_event<256, false, false>);
}

// DP: construct the per-universe tracker objects (objs: n_univ * kTrkBytes, tab: n_univ pointers)
cudaError_t dp_init(const DevGeom& g, void* objs, void* tab, cudaStream_t stream) {
  k_dp_init<<<(g.n_univ + 127) / 128, 128, 0, stream>>>(g, static_cast<unsigned char*>(objs),
                                                         static_cast<const void**>(tab));
  return cudaGetLastError();
}
size_t dp_object_bytes() { return kTrkBytes; }

cudaError_t launch_wq(const DevGeom& g, const KRun& R, bool trace, bool states, int blocks_per_sm,
                      cudaStream_t stream, int* grid_out) {
  const size_t smem = wq_smem_bytes(g, trace);
  const int block = kWqWarps * 32;
  auto go = [&](auto kern) -> cudaError_t {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int dev = 0, nsm = 0, occ = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, block, smem);
    if (e != cudaSuccess) return e;
    if (occ < 1) return cudaErrorInvalidConfiguration;
    const int bps = blocks_per_sm > 0 ? (blocks_per_sm < occ ? blocks_per_sm : occ) : occ;
    const uint64_t per_block = (uint64_t)kWqWarps * kWqSlots;
    uint64_t need = (R.n + per_block - 1) / per_block, grid = (uint64_t)nsm * bps;
    if (need < grid) grid = need ? need : 1;
    *grid_out = (int)grid;
    return with_slices(g, R, grid, stream, [&](const KRun& Rs) {
      kern<<<(unsigned)grid, block, smem, stream>>>(g, Rs);
      return cudaGetLastError();
    });
  };
  const int tally = (R.mesh ? 1 : 0) | (R.inst ? 2 : 0);
  if (tally) {
    if (trace) return cudaErrorNotSupported;
    if (tally == 1) return states ? go(k_track_wq<false, true, 1>) : go(k_track_wq<false, false, 1>);
    if (tally == 2) return states ? go(k_track_wq<false, true, 2>) : go(k_track_wq<false, false, 2>);
    return states ? go(k_track_wq<false, true, 3>) : go(k_track_wq<false, false, 3>);
  }
  if (trace) return states ? go(k_track_wq<true, true>) : go(k_track_wq<true, false>);
  return states ? go(k_track_wq<false, true>) : go(k_track_wq<false, false>);
}

// device self-test: fdiv / fsqrt against IEEE `/` and sqrt on operands spanning the walk's ranges
__global__ void k_selftest_arith(uint64_t n, uint64_t seed, unsigned long long* bad) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    double x0, x1, x2, x3;
    draw2(seed, i, 7, 0, x0, x1);
    draw2(seed, i, 7, 1, x2, x3);
    double a = exp10(-20.0 + 26.0 * x0) * (x1 < 0.5 ? -1.0 : 1.0);
    if (x1 > 0.98) a = 0.0;
    const double b = exp10(-25.0 + 25.5 * x2) * (x3 < 0.5 ? -1.0 : 1.0);
    const double xs = x3 > 0.99 ? 0.0 : exp10(-40.0 + 52.0 * x0);
    const double q1 = fdiv(a, b), q2 = a / b;
    if (__double_as_longlong(q1) != __double_as_longlong(q2)) atomicAdd(bad, 1ull);
    const double s1 = fsqrt(xs), s2 = sqrt(xs);
    if (__double_as_longlong(s1) != __double_as_longlong(s2)) atomicAdd(bad + 1, 1ull);
    // geometric shapes: differences of nearby coordinates over direction cosines
    const double e = (x2 - 0.5) * 400.0, xx = e + (x0 - 0.5) * 1e-6;
    const double q3 = fdiv(e - xx, x1 - 0.5), q4 = (e - xx) / (x1 - 0.5);
    if (__double_as_longlong(q3) != __double_as_longlong(q4)) atomicAdd(bad, 1ull);
  }
}

// ---------------------------------------------------------------- F1: next-cycle fission source
// exclusive prefix of the per-history site counts (three passes: block sums, one-block scan of
// the sums, per-element prefix), then one thread per source particle: flat site index
// floor(u * M), binary search for its history, isotropic direction (see nt_fission_source).
constexpr int kScanB = 1024;

__global__ void __launch_bounds__(kScanB) k_bank_block_sums(const uint8_t* bn, uint64_t n, unsigned long long* sums) {
  __shared__ unsigned long long sh[kScanB / 32];
  const uint64_t i = blockIdx.x * (uint64_t)kScanB + threadIdx.x;
  unsigned long long v = i < n ? bn[i] : 0ull;
  for (int o = 16; o; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long t = 0;
    for (int k = 0; k < kScanB / 32; ++k) t += sh[k];
    sums[blockIdx.x] = t;
  }
}

__global__ void k_bank_scan_sums(unsigned long long* sums, uint64_t nb, unsigned long long* total) {
  if (threadIdx.x != 0) return;                       // nb <= ~1e5: one thread is plenty
  unsigned long long acc = 0;
  for (uint64_t b = 0; b < nb; ++b) { const unsigned long long v = sums[b]; sums[b] = acc; acc += v; }
  *total = acc;
}

__global__ void __launch_bounds__(kScanB) k_bank_prefix(const uint8_t* bn, uint64_t n, const unsigned long long* offs,
                                                        unsigned long long* prefix) {
  __shared__ unsigned long long sh[kScanB / 32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint64_t i = blockIdx.x * (uint64_t)kScanB + threadIdx.x;
  const unsigned long long v = i < n ? bn[i] : 0ull;
  unsigned long long x = v;                           // inclusive warp scan
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) sh[w] = x;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long acc = 0;
    for (int k = 0; k < kScanB / 32; ++k) { const unsigned long long t = sh[k]; sh[k] = acc; acc += t; }
  }
  __syncthreads();
  if (i < n) prefix[i] = offs[blockIdx.x] + sh[w] + (x - v);
}

// flat (history, site)-ordered site list: sites[(prefix[i] + k) * 3 + a]
__global__ void k_bank_compact(const double* bank, const uint8_t* bn, const unsigned long long* prefix, uint64_t n,
                               int ms, double* sites) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const int c = bn[i];
    for (int k = 0; k < c; ++k)
      for (int a = 0; a < 3; ++a) sites[(prefix[i] + k) * 3 + a] = bank[(i * ms + k) * 3 + a];
  }
}

// source particle J = j_begin + j: site floor(u_J * M) of the flat list, isotropic direction
__global__ void k_source_from_sites(const double* sites, unsigned long long M, uint64_t seed, uint32_t cycle,
                                    uint64_t j_begin, uint64_t n_next, double* st) {
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < n_next; j += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t J = j_begin + j;
    double u, unused, xmu, xphi, ox, oy, oz;
    draw2(seed, J, cycle, 0xF155u, u, unused);
    const unsigned long long t = static_cast<unsigned long long>(floor(u * static_cast<double>(M)));
    const double* p = sites + t * 3;
    draw2(seed, J, cycle, 0xF156u, xmu, xphi);
    isotropic(xmu, xphi, ox, oy, oz);
    st[j] = p[0]; st[n_next + j] = p[1]; st[2 * n_next + j] = p[2];
    st[3 * n_next + j] = ox; st[4 * n_next + j] = oy; st[5 * n_next + j] = oz;
  }
}

static unsigned grid_for(uint64_t n) {
  uint64_t grid = (n + 255) / 256;
  if (grid > 148 * 16) grid = 148 * 16;
  return (unsigned)(grid ? grid : 1);
}

cudaError_t bank_compact(const DevGeom& g, const double* bank, const uint8_t* bank_n, uint64_t n, double* sites,
                         unsigned long long* M_host, cudaStream_t stream) {
  *M_host = 0;
  if (n == 0) return cudaSuccess;
  const uint64_t nb = (n + kScanB - 1) / kScanB;
  unsigned long long* scratch = nullptr;             // sums[nb] | total | prefix[n]
  cudaError_t e = scratch_alloc(g, &scratch, (nb + 1 + n) * sizeof(unsigned long long), stream);
  if (e != cudaSuccess) return e;
  unsigned long long *sums = scratch, *total = scratch + nb, *prefix = scratch + nb + 1;
  k_bank_block_sums<<<(unsigned)nb, kScanB, 0, stream>>>(bank_n, n, sums);
  k_bank_scan_sums<<<1, 32, 0, stream>>>(sums, nb, total);
  k_bank_prefix<<<(unsigned)nb, kScanB, 0, stream>>>(bank_n, n, sums, prefix);
  k_bank_compact<<<grid_for(n), 256, 0, stream>>>(bank, bank_n, prefix, n, g.max_sites, sites);
  e = cudaMemcpyAsync(M_host, total, sizeof(unsigned long long), cudaMemcpyDeviceToHost, stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
  const cudaError_t e2 = cudaFreeAsync(scratch, stream);
  return e != cudaSuccess ? e : e2;
}

cudaError_t source_from_sites(const double* sites, unsigned long long M, uint64_t seed, uint32_t cycle,
                              uint64_t j_begin, uint64_t n_next, double* states, cudaStream_t stream) {
  if (M == 0 || n_next == 0) return cudaSuccess;
  k_source_from_sites<<<grid_for(n_next), 256, 0, stream>>>(sites, M, seed, cycle, j_begin, n_next, states);
  return cudaGetLastError();
}

cudaError_t fission_source(const DevGeom& g, const double* bank, const uint8_t* bank_n, uint64_t n_prev,
                           uint64_t seed, uint32_t cycle, uint64_t n_next, double* states,
                           unsigned long long* M_host, cudaStream_t stream) {
  *M_host = 0;
  if (n_prev == 0) return cudaSuccess;
  double* sites = nullptr;
  cudaError_t e = scratch_alloc(g, &sites, n_prev * (uint64_t)g.max_sites * 3 * sizeof(double), stream);
  if (e != cudaSuccess) return e;
  e = bank_compact(g, bank, bank_n, n_prev, sites, M_host, stream);
  if (e == cudaSuccess) e = source_from_sites(sites, *M_host, seed, cycle, 0, n_next, states, stream);
  const cudaError_t e2 = cudaFreeAsync(sites, stream);
  return e != cudaSuccess ? e : e2;
}

cudaError_t bih_stats(unsigned long long* host4, bool reset) {
#ifdef NT_BIH_STATS
  if (reset) { unsigned long long z[16] = {}; return cudaMemcpyToSymbol(g_bih_stats, z, sizeof z); }
  return cudaMemcpyFromSymbol(host4, g_bih_stats, 16 * sizeof(unsigned long long));
#else
  (void)host4; (void)reset;
  return cudaErrorNotSupported;
#endif
}

cudaError_t selftest_arith(uint64_t n, uint64_t seed, unsigned long long* d_bad) {
  k_selftest_arith<<<148 * 8, 256>>>(n, seed, d_bad);
  return cudaGetLastError();
}

cudaError_t launch_find_cells(const DevGeom& g, const double* xyz, uint64_t n, int32_t* cell,
                              uint8_t* flag, cudaStream_t stream) {
  const int block = 256;
  const size_t smem = (size_t)block * ((g.max_depth - 1) * 3 * 8 + g.max_depth * 4 * 4);
  cudaError_t e = cudaFuncSetAttribute(k_find_cells, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  uint64_t grid = (n + block - 1) / block;
  if (grid > 148 * 8) grid = 148 * 8;
  if (grid == 0) return cudaSuccess;
  k_find_cells<<<(unsigned)grid, block, smem, stream>>>(g, xyz, n, cell, flag);
  return cudaGetLastError();
}

#endif  // NT_RECT_TU
NT_DEV_END
