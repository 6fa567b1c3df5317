// Device geometry primitives for the generic tracker (sm_100a, fp64, -fmad=false):
// implicit functions and senses (readings O3/O4), cell-aware forward distances
// (Table 1 distance_to_surface, reading O11), BIH point location, rect
// (Alg. 5-6) and hex (reading O9) tile location, and the per-level distance candidates.
#pragma once
#include <cstdint>

#include "nt_layout.hpp"
#include "nt_math.cuh"

NT_DEV_BEGIN

#define NT_INF __longlong_as_double(0x7ff0000000000000ULL)

// kinds compiled into this feature set (see nt_layout.hpp)
constexpr bool kHex = (NT_FEAT & F_HEX) != 0;
constexpr bool kPlane = (NT_FEAT & F_PLANE) != 0;
constexpr bool kSphere = (NT_FEAT & F_SPHERE) != 0;
constexpr bool kRectNU = (NT_FEAT & F_RECTNU) != 0;

template <class T>
__device__ __forceinline__ T ld(const T* p) { return __ldg(p); }

// d > 0 ? d : 0 as one compare and one select (nvcc otherwise emits a NaN-propagating max sequence;
// the result is the same for every input, NaN -> 0 included)
__device__ __forceinline__ double clamp0(double d) {
  double r;
  asm("{\n\t.reg .pred p;\n\tsetp.gt.f64 p, %1, 0d0000000000000000;\n\tselp.f64 %0, %1, 0d0000000000000000, p;\n\t}"
      : "=d"(r) : "d"(d));
  return r;
}

// p ? a : b as one predicated select (no branch)
__device__ __forceinline__ double dsel(bool p, double a, double b) {
  double r;
  asm("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %3, 0;\n\tselp.f64 %0, %1, %2, q;\n\t}"
      : "=d"(r) : "d"(a), "d"(b), "r"(static_cast<unsigned>(p)));
  return r;
}
__device__ __forceinline__ double sel3(int a, double x, double y, double z) {
  return dsel(a == 0, x, dsel(a == 1, y, z));
}

// f(r) of a surface (O3), evaluation order exactly as documented
__device__ __forceinline__ double surf_f(int kind, const double* sp, double x, double y, double z) {
  if (kind <= S_PZ) return sel3(kind, x, y, z) - ld(&sp[0]);
  const double c0 = ld(&sp[0]), c1 = ld(&sp[1]), c2 = ld(&sp[2]), c3 = ld(&sp[3]);
  if (kPlane && kind == S_PLANE) return ((c0 * x + c1 * y) + c2 * z) - c3;
  const double dx = x - c0, dy = y - c1;
  if (!kSphere || kind == S_CZ) return (dx * dx + dy * dy) - c2;
  const double dz = z - c2;
  return ((dx * dx + dy * dy) + dz * dz) - c3;
}

// forward distance to leave half-space (kind, sense) along (u,v,w) from (x,y,z); O11.
// os: particle logically on this surface (quadric c := 0).  Returns +inf when no exit.
// Written with ONE division and ONE square root per call (selected operands) to keep the
// code small; the selected operands are exactly those of the case formulas in DESIGN.md O11.
// Coefficients are passed by value: the caller loads the whole record before the kind branch, so
// the loads overlap (surf_dist(..., const double* sp, ...) below loads them for other callers).
__device__ __forceinline__ double surf_dist(int kind, int sense, bool os, double c0, double c1, double c2,
                                            double c3, double x, double y, double z, double u, double v,
                                            double w) {
  double num, den;
  bool ok;
  if (kind <= S_PZ) {
    den = sel3(kind, u, v, w);
    ok = sense ? den < 0.0 : den > 0.0;                      // also excludes den == 0
    num = c0 - sel3(kind, x, y, z);
  } else {
    if (kPlane && kind == S_PLANE) {
      den = (c0 * u + c1 * v) + c2 * w;
      ok = sense ? den < 0.0 : den > 0.0;
      num = c3 - ((c0 * x + c1 * y) + c2 * z);
    } else {
      double a, k, c, q;
      if (!kSphere || kind == S_CZ) {
        const double dx = x - c0, dy = y - c1;
        a = u * u + v * v;
        k = dx * u + dy * v;
        c = os ? 0.0 : (dx * dx + dy * dy) - c2;
        q = k * k - a * c;
      } else {
        const double dx = x - c0, dy = y - c1, dz = z - c2;
        a = 1.0;
        k = (dx * u + dy * v) + dz * w;
        c = os ? 0.0 : ((dx * dx + dy * dy) + dz * dz) - c3;
        q = k * k - c;
      }
      const double sq = fsqrt(clamp0(q));                 // q < 0: max(q,0) inside, miss outside
      // inside (negative side), far root: k <= 0 -> (-k + sq) / a, else -c / (k + sq);
      // outside: c / (-k + sq), no exit when moving away or missing.  Operands by selects.
      const bool far = !sense && k <= 0.0;
      const double mk = dsel(sense, -k, k);                // den = mk + sq unless `far`
      num = dsel(far, -k + sq, dsel(sense, c, -c));
      den = dsel(far, a, mk + sq);
      ok = a != 0.0 && (!sense || (k < 0.0 && q >= 0.0));
    }
  }
  // the division runs on every lane (a lane without a forward exit would idle beside the others
  // anyway); its result is discarded by the select
  return dsel(ok, clamp0(fdiv(num, den)), NT_INF);
}
__device__ __forceinline__ double surf_dist(int kind, int sense, bool os, const double* sp, double x,
                                            double y, double z, double u, double v, double w) {
  return surf_dist(kind, sense, os, ld(&sp[0]), ld(&sp[1]), ld(&sp[2]), ld(&sp[3]), x, y, z, u, v, w);
}

// Alg. 3 "cell contains pos" with an optional logically forced sense (O9'); on success the
// O16 F1 proximity bit of the accepted cell is returned in `near`.
__device__ __forceinline__ bool cell_contains(const DevGeom& g, int h0, int h1, double x, double y, double z,
                                              int fsid, int fsense, uint32_t& near) {
  uint32_t nb = 0;
  for (int h = h0; h < h1; ++h) {
    const DHs* r = g.hsr + h;
    const int e = ld(&r->e);
    const int sid = hs_sid(e);
    int s;
    if (sid == fsid) {
      s = fsense;
    } else {
      const double f = surf_f(hs_kind(e), r->c, x, y, z);
      s = f >= 0.0;
      if (fabs(f) <= ld(&r->tol)) nb = 1u;
    }
    if (s != hs_sense(e)) return false;
  }
  near = nb;
  return true;
}

// BIH traversal for point location: both children are visited when the point lies
// in their overlap.  Register-resident stack: up to kBihStack pending node indices (relative to the
// universe's root, 16 bits each) packed in three 64-bit registers -- no local memory.  The builder
// bounds the tree depth by kBihStack and the node count per universe by 65536, so the stack
// cannot overflow.  "While-while" form: a lane first walks internal nodes down to a leaf, then
// tests the leaf's cells, which keeps the lanes of a warp on the same loop body.
struct BihStack {
  uint64_t s0 = 0, s1 = 0, s2 = 0;
  __device__ __forceinline__ void push(uint32_t v) {
    s2 = (s2 << 16) | (s1 >> 48);
    s1 = (s1 << 16) | (s0 >> 48);
    s0 = (s0 << 16) | v;
  }
  // returns the popped index, or -1 when empty (entries are stored +1 so that 0 marks empty)
  __device__ __forceinline__ int pop() {
    const int v = static_cast<int>(s0 & 0xFFFFull) - 1;
    s0 = (s0 >> 16) | (s1 << 48);
    s1 = (s1 >> 16) | (s2 << 48);
    s2 >>= 16;
    return v;
  }
};

#ifdef NT_BIH_STATS
// calls, node visits, cell tests, -, max cells / call, max nodes / call, [6..15] log2 histogram of cells / call
__device__ unsigned long long g_bih_stats[16];
__device__ __forceinline__ void bih_stats_done(unsigned cells, unsigned nodes) {
  atomicMax(&g_bih_stats[4], (unsigned long long)cells);
  atomicMax(&g_bih_stats[5], (unsigned long long)nodes);
  const int b = cells ? min(9, 32 - __clz(cells)) : 0;
  atomicAdd(&g_bih_stats[6 + b], 1ull);
}
#endif
// `first` / `nfirst`: an optional list of cells tested before the search (the crossing shortcut's
// neighbours across the crossed half-space).  It is run as a leaf whose continuation is the root, so
// the kernel holds one copy of the containment test.
// Returns the cell (or -1) and its fill in `fill`.
__device__ __forceinline__ int csg_find(const DevGeom& g, int root, double x, double y, double z,
                                        int fsid, int fsense, uint32_t& flags, int& fill, int& h0, int& h1,
                                        const CRef* first = nullptr, int nfirst = 0) {
#ifdef NT_BIH_STATS
  atomicAdd(&g_bih_stats[0], 1ull);
#endif
  BihStack stk;
  int node = 0;                                          // relative to root
  bool pre = nfirst > 0;
  if (pre) stk.push(1u);                                 // after the list: the root (stored +1)
#ifdef NT_BIH_STATS
  unsigned st_cells = 0, st_nodes = 0;
#define NT_BIH_RET(v) do { bih_stats_done(st_cells, st_nodes); return (v); } while (0)
#else
#define NT_BIH_RET(v) return (v)
#endif
  for (;;) {
    int meta = 0, a = 0;
    const CRef* leaf = first;
    for (; !pre;) {                                      // internal nodes down to a leaf
      const BihNode* n = g.bih + root + node;
      meta = ld(&n->meta);
      a = ld(&n->a);
#ifdef NT_BIH_STATS
      atomicAdd(&g_bih_stats[1], 1ull);
      ++st_nodes;
#endif
      if (meta < 0) break;
      const double c = sel3(meta, x, y, z);
      const bool gl = c <= ld(&n->lmax), gr = c >= ld(&n->rmin);
      const int left = a - root;
      if (gl && gr) { stk.push(static_cast<uint32_t>(left + 2)); node = left; }
      else if (gl) node = left;
      else if (gr) node = left + 1;
      else {
        node = stk.pop();
        if (node < 0) NT_BIH_RET(-1);
      }
    }
    int cnt = nfirst;
    if (!pre) { leaf = g.bih_leaf + a; cnt = -meta - 1; }   // leaf: test its cells
    pre = false;
    for (int q = 0; q < cnt; ++q) {
      const int4 cr = __ldg(reinterpret_cast<const int4*>(leaf + q));   // cell, fill, h0, h1
      uint32_t nb = 0;
#ifdef NT_BIH_STATS
      atomicAdd(&g_bih_stats[2], 1ull);
      ++st_cells;
#endif
      if (cell_contains(g, cr.z, cr.w, x, y, z, fsid, fsense, nb)) {
        flags |= nb;
        fill = cr.y;
        h0 = cr.z;
        h1 = cr.w;
        NT_BIH_RET(cr.x);
      }
    }
    node = stk.pop();
    if (node < 0) NT_BIH_RET(-1);
  }
#undef NT_BIH_RET
}

// forward wall of a rect tile along one axis (O11 RECT walls): (e(i+1) - x)/u or (e(i) - x)/u
__device__ __forceinline__ double rect_wall(double ll, double p, int i, double x, double u) {
  const double e = ll + static_cast<double>(u > 0.0 ? i + 1 : i) * p;
  return clamp0(fdiv(e - x, u));
}

// O8: the unique i with e(i) <= x < e(i+1), e(i) = ll + i p
__device__ __forceinline__ int rect_index(double ll, double p, double x) {
  int i = static_cast<int>(floor(fdiv(x - ll, p)));
  while (!(ll + static_cast<double>(i) * p <= x)) --i;
  while (!(x < ll + static_cast<double>(i + 1) * p)) ++i;
  return i;
}

__device__ __forceinline__ bool near_wall(double ll, double p, int i, double x) {
  return fabs(x - (ll + static_cast<double>(i) * p)) <= kFlagDist ||
         fabs(x - (ll + static_cast<double>(i + 1) * p)) <= kFlagDist;
}

// Distance-to-boundary bookkeeping: strict '<' keeps the top-most level / lowest id on exact
// ties (O13); d2 = smallest other candidate (O16 F2).
// The winner is packed in one register (level | sense << 4 | surface-or-face << 5) so that the
// select form costs one integer select, and +inf candidates are harmless no-ops.
struct Best {
  double d, d2;
  int key;
  __device__ __forceinline__ void init() { d = NT_INF; d2 = NT_INF; key = -1; }
  __device__ __forceinline__ int l() const { return key & 15; }
  __device__ __forceinline__ int sense() const { return (key >> 4) & 1; }
  __device__ __forceinline__ int j() const { return key >> 5; }
  // p ? a : b as one predicated select (keeps the candidate loop branch-free)
  static __device__ __forceinline__ double selp(double a, double b, bool p) {
    double r;
    asm("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %3, 0;\n\tselp.f64 %0, %1, %2, q;\n\t}"
        : "=d"(r) : "d"(a), "d"(b), "r"(static_cast<unsigned>(p)));
    return r;
  }
  __device__ __forceinline__ void consider(double dd, int ll, int jj, int ss) {
    const bool lt = dd < d;                       // min / second-min, branch-free
    const double hi = selp(d, dd, lt);            // the larger of (d, dd)
    d = selp(dd, d, lt);
    d2 = selp(hi, d2, hi < d2);
    key = lt ? (ll | (ss << 4) | (jj << 5)) : key;
  }
};

// ---- F1 fission bank: an absorption in material cell mc banks floor(nut + xi) sites at the
// absorption point (xi = the collision draw's second uniform, unused by an absorption).
__device__ __forceinline__ void bank_sites(const DevGeom& g, double* bank, uint8_t* bank_n, int mc, uint64_t idx,
                                           double xi, double x, double y, double z) {
  const double nut = ld(g.mc_nut + mc);
  if (!(nut > 0.0)) return;
  int ns = static_cast<int>(floor(nut + xi));
  if (ns > g.max_sites) ns = g.max_sites;
  double* p = bank + idx * static_cast<uint64_t>(g.max_sites) * 3;
  for (int k = 0; k < ns; ++k) { p[3 * k] = x; p[3 * k + 1] = y; p[3 * k + 2] = z; }
  bank_n[idx] = static_cast<uint8_t>(ns);
}

// ---- superimposed mesh track-length tally (NEXT-2; reading M1).  3-D DDA along the
// segment r + t om, t in [0, s].  The cut parameters are (E_a(i) - r_a) / om_a with
// E_a(i) = lo_a + i d_a -- the oracle's -- so every scored piece is the oracle's piece.  Pieces
// outside the mesh are skipped; the walk stops once the ray leaves the mesh on some axis.
// Inlined: only the mesh-tally kernel instantiations (TALLY & 1) contain the call.
struct MeshGeom { double lo[3], d[3]; int n[3]; };

__device__ __forceinline__ void mesh_score_impl(const MeshGeom M, double* out, double x, double y, double z,
                                             double u, double v, double w, double s) {
  if (!(s > 0.0)) return;
  const double r[3] = {x, y, z}, om[3] = {u, v, w};
  int idx[3];
  double tn[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const double lo = M.lo[a], d = M.d[a];
    int i = rect_index(lo, d, r[a]);                             // E(i) <= r < E(i+1)
    if (om[a] < 0.0 && r[a] == lo + static_cast<double>(i) * d) --i;   // on a plane, moving down
    idx[a] = i;
    tn[a] = om[a] > 0.0 ? fdiv(lo + static_cast<double>(i + 1) * d - r[a], om[a])
          : om[a] < 0.0 ? fdiv(lo + static_cast<double>(i) * d - r[a], om[a]) : NT_INF;
  }
  const int n0 = M.n[0], n1 = M.n[1], n2 = M.n[2];
  double t = 0.0;
#pragma unroll 1
  for (;;) {
    if ((idx[0] < 0 && !(u > 0.0)) || (idx[0] >= n0 && !(u < 0.0)) || (idx[1] < 0 && !(v > 0.0)) ||
        (idx[1] >= n1 && !(v < 0.0)) || (idx[2] < 0 && !(w > 0.0)) || (idx[2] >= n2 && !(w < 0.0)))
      return;                                                    // left the mesh for good
    const double te = fmin(fmin(tn[0], tn[1]), fmin(tn[2], s));
    const bool in = idx[0] >= 0 && idx[0] < n0 && idx[1] >= 0 && idx[1] < n1 && idx[2] >= 0 && idx[2] < n2;
    if (in && te > t) atomicAdd(out + idx[0] + n0 * (idx[1] + n1 * idx[2]), te - t);
    if (te >= s) return;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      if (tn[a] == te) {
        const double lo = M.lo[a], d = M.d[a];
        if (om[a] > 0.0) {
          ++idx[a];
          tn[a] = fdiv(lo + static_cast<double>(idx[a] + 1) * d - r[a], om[a]);
        } else {
          --idx[a];
          tn[a] = fdiv(lo + static_cast<double>(idx[a]) * d - r[a], om[a]);
        }
      }
    }
    t = te;
  }
}

__device__ __forceinline__ void mesh_score(const DevGeom& g, double* out, double x, double y, double z, double u,
                                           double v, double w, double s) {
  MeshGeom M;
  for (int a = 0; a < 3; ++a) { M.lo[a] = g.mesh_lo[a]; M.d[a] = g.mesh_d[a]; M.n[a] = g.mesh_n[a]; }
  mesh_score_impl(M, out, x, y, z, u, v, w, s);
}

// ---- non-uniform rect arrays (reading N1; Alg. 5 binary search over the mesh divisions,
// P:500-525).  Axis divisions e[0..n]; tile -1 is the slab below e[0], tile n the slab at or
// above e[n] (both `outer`); the slabs have no wall on their open side.
__device__ __forceinline__ int nu_index(const double* e, int n, double x) {
  if (x < ld(e)) return -1;
  if (!(x < ld(e + n))) return n;
  int lo = 0, hi = n;                                   // e[lo] <= x < e[hi]
#pragma unroll 1
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (ld(e + mid) <= x) lo = mid; else hi = mid;
  }
  return lo;
}
__device__ __forceinline__ bool nu_near(const double* e, int n, int i, double x) {
  return (i >= 0 && fabs(x - ld(e + i)) <= kFlagDist) || (i + 1 <= n && fabs(x - ld(e + i + 1)) <= kFlagDist);
}
__device__ __forceinline__ double nu_wall(const double* e, int n, int i, double x, double u) {
  const int k = u > 0.0 ? i + 1 : i;
  if (k < 0 || k > n) return NT_INF;
  return clamp0(fdiv(ld(e + k) - x, u));
}
__device__ __forceinline__ double nu_centre(const double* e, int n, int i) {
  if (i < 0) return ld(e);
  if (i >= n) return ld(e + n);
  return (ld(e + i) + ld(e + i + 1)) * 0.5;
}

// Alg. 5 find_cell at a rect level: tile (i, j, k) of the local point, F1 proximity flags
__device__ __forceinline__ void rect_locate(const DevGeom& g, const DUniv* U, double x, double y, double z,
                                            int& i, int& j, int& k, uint32_t& flags) {
  const int is2d = ld(&U->is2d);
  if (kRectNU) {
    const int eo = ld(&U->ntile);
    if (eo >= 0) {
      const int n0 = ld(&U->i0), n1 = ld(&U->i1);
      const double* ex = g.edges + eo;
      const double* ey = ex + n0 + 1;
      i = nu_index(ex, n0, x);
      j = nu_index(ey, n1, y);
      k = 0;
      uint32_t nb = nu_near(ex, n0, i, x) | nu_near(ey, n1, j, y);
      if (!is2d) {
        const int n2 = ld(&U->i2);
        const double* ez = ey + n1 + 1;
        k = nu_index(ez, n2, z);
        nb |= nu_near(ez, n2, k, z);
      }
      flags |= nb;
      return;
    }
  }
  const double llx = ld(&U->d[0]), lly = ld(&U->d[1]), px = ld(&U->d[3]), py = ld(&U->d[4]);
  i = rect_index(llx, px, x);
  j = rect_index(lly, py, y);
  uint32_t nb = near_wall(llx, px, i, x) | near_wall(lly, py, j, y);
  k = 0;
  if (!is2d) {
    const double llz = ld(&U->d[2]), pz = ld(&U->d[5]);
    k = rect_index(llz, pz, z);
    nb |= near_wall(llz, pz, k, z);
  }
  flags |= nb;
}

// distance_to_boundary candidates of rect tile (ia, ib, ic) at level l (forward walls, O11)
__device__ __forceinline__ void rect_candidates(const DevGeom& g, const DUniv* U, int ia, int ib, int ic, int l,
                                                double x, double y, double z, double u, double v, double w,
                                                Best& b) {
  if (kRectNU) {
    const int eo = ld(&U->ntile);
    if (eo >= 0) {
      const int n0 = ld(&U->i0), n1 = ld(&U->i1);
      const double* ex = g.edges + eo;
      const double* ey = ex + n0 + 1;
      if (u != 0.0) b.consider(nu_wall(ex, n0, ia, x, u), l, u > 0.0 ? 1 : 0, 0);
      if (v != 0.0) b.consider(nu_wall(ey, n1, ib, y, v), l, v > 0.0 ? 3 : 2, 0);
      if (!ld(&U->is2d) && w != 0.0) b.consider(nu_wall(ey + n1 + 1, ld(&U->i2), ic, z, w), l, w > 0.0 ? 5 : 4, 0);
      return;
    }
  }
  // an axis with a zero direction cosine has no wall: +inf (a no-op for consider), selected, no branch
  b.consider(dsel(u != 0.0, rect_wall(ld(&U->d[0]), ld(&U->d[3]), ia, x, u), NT_INF), l, u > 0.0 ? 1 : 0, 0);
  b.consider(dsel(v != 0.0, rect_wall(ld(&U->d[1]), ld(&U->d[4]), ib, y, v), NT_INF), l, v > 0.0 ? 3 : 2, 0);
  if (!ld(&U->is2d))
    b.consider(dsel(w != 0.0, rect_wall(ld(&U->d[2]), ld(&U->d[5]), ic, z, w), NT_INF), l, w > 0.0 ? 5 : 4, 0);
}

// tile centre of an array (the daughter translation, readings O8/O9/N1).  rect (i,j,k), hex (q,r,kz).
__device__ __forceinline__ void array_centre(const DevGeom& g, const DUniv* U, int kind, int a, int b, int c,
                                             double& tx, double& ty, double& tz) {
  if (kRectNU && kind == U_RECT && ld(&U->ntile) >= 0) {
    const int n0 = ld(&U->i0), n1 = ld(&U->i1);
    const double* ex = g.edges + ld(&U->ntile);
    const double* ey = ex + n0 + 1;
    tx = nu_centre(ex, n0, a);
    ty = nu_centre(ey, n1, b);
    tz = ld(&U->is2d) ? 0.0 : nu_centre(ey + n1 + 1, ld(&U->i2), c);
    return;
  }
  if (!kHex || kind == U_RECT) {
    tx = ld(&U->d[0]) + (static_cast<double>(a) + 0.5) * ld(&U->d[3]);
    ty = ld(&U->d[1]) + (static_cast<double>(b) + 0.5) * ld(&U->d[4]);
    tz = ld(&U->is2d) ? 0.0 : ld(&U->d[2]) + (static_cast<double>(c) + 0.5) * ld(&U->d[5]);
  } else {
    tx = ld(&U->d[0]) + (static_cast<double>(a) * ld(&U->d[6]) + static_cast<double>(b) * ld(&U->d[8]));
    ty = ld(&U->d[1]) + (static_cast<double>(a) * ld(&U->d[7]) + static_cast<double>(b) * ld(&U->d[9]));
    tz = ld(&U->i1) > 0 ? ld(&U->d[4]) + (static_cast<double>(c) + 0.5) * ld(&U->d[5]) : 0.0;
  }
}

// daughter universe of an array tile (fill inside the lattice, else outer) and the tile
// centre (daughter translation).  Tile indices: rect (i,j,k), hex (q,r,kz).
__device__ __forceinline__ int array_daughter(const DevGeom& g, const DUniv* U, int kind, int a, int b,
                                              int c, double& tx, double& ty, double& tz) {
  int idx = -1;
  if (!kHex || kind == U_RECT) {
    const int n0 = ld(&U->i0), n1 = ld(&U->i1), n2 = ld(&U->i2), is2d = ld(&U->is2d);
    const bool in = a >= 0 && a < n0 && b >= 0 && b < n1 && (is2d || (c >= 0 && c < n2));
    if (in) idx = ld(g.fills + ld(&U->fill_off) + a + n0 * (b + n1 * (is2d ? 0 : c)));
  } else {
    const int R = ld(&U->i0), nz = ld(&U->i1);
    const int aq = abs(a), ar = abs(b), as = abs(a + b);
    const int dd = max(aq, max(ar, as));
    const bool in = dd <= R && (nz == 0 || (c >= 0 && c < nz));
    if (in) idx = ld(g.fills + ld(&U->fill_off) + (b + R) * (2 * R + 1) + (a + R) + (nz > 0 ? c * ld(&U->ntile) : 0));
  }
  array_centre(g, U, kind, a, b, c, tx, ty, tz);
  return idx >= 0 ? idx : ld(&U->outer);
}

// hex s-space coordinates s_k = n_k . (x - C) (reading O9): tile (q, r) spans
// p (m_k - 1/2) <= s_k < p (m_k + 1/2); no division
__device__ __forceinline__ void hex_t(const DUniv* U, double x, double y, double& t0, double& t1, double& t2) {
  const double xp = x - ld(&U->d[0]), yp = y - ld(&U->d[1]);
  t0 = ld(&U->d[10]) * xp + ld(&U->d[11]) * yp;
  t1 = ld(&U->d[12]) * xp + ld(&U->d[13]) * yp;
  t2 = ld(&U->d[14]) * xp + ld(&U->d[15]) * yp;
}

__device__ __forceinline__ void hex_m(int q, int r, double& m0, double& m1, double& m2) {
  const double qd = static_cast<double>(q), rd = static_cast<double>(r);
  m0 = qd + rd * 0.5;
  m1 = qd * 0.5 + rd;
  m2 = -(qd * 0.5) + rd * 0.5;
}

// hex tile owning (x,y): cube rounding then fix-up moves in s-space (O9); falls back to the
// cube-rounded tile with F1 if the fix-up does not converge.  Sets F1 on proximity.
__device__ __forceinline__ void hex_locate(const DUniv* U, double x, double y, int& qo, int& ro, uint32_t& flags) {
  const double xp = x - ld(&U->d[0]), yp = y - ld(&U->d[1]);
  const double p = ld(&U->d[2]), pH = ld(&U->d[3]);
  double qf, rf;
  if (ld(&U->i2) == 0) { rf = fdiv(yp, pH); qf = fdiv(xp - rf * (p * 0.5), p); }
  else { qf = fdiv(xp, pH); rf = fdiv(yp - qf * (p * 0.5), p); }
  const double sf = -qf - rf;
  double qr = round(qf), rr = round(rf), sr = round(sf);
  const double dq = fabs(qr - qf), dr = fabs(rr - rf), ds = fabs(sr - sf);
  if (dq > dr && dq > ds) qr = -rr - sr;
  else if (dr > ds) rr = -qr - sr;
  const int qc = static_cast<int>(qr), rc = static_cast<int>(rr);
  double t0, t1, t2;
  hex_t(U, x, y, t0, t1, t2);
  int q = qc, r = rc;
  bool ok = false;
#pragma unroll 1
  for (int it = 0; it < 4; ++it) {
    double m0, m1, m2;
    hex_m(q, r, m0, m1, m2);
    if (t0 < p * (m0 - 0.5)) { q -= 1; continue; }            // face 3: delta (-1, 0)
    if (!(t0 < p * (m0 + 0.5))) { q += 1; continue; }         // face 0: delta (+1, 0)
    if (t1 < p * (m1 - 0.5)) { r -= 1; continue; }            // face 4: delta (0, -1)
    if (!(t1 < p * (m1 + 0.5))) { r += 1; continue; }         // face 1: delta (0, +1)
    if (t2 < p * (m2 - 0.5)) { q += 1; r -= 1; continue; }    // face 5: delta (+1, -1)
    if (!(t2 < p * (m2 + 0.5))) { q -= 1; r += 1; continue; } // face 2: delta (-1, +1)
    ok = true;
    break;
  }
  if (!ok) { q = qc; r = rc; flags |= 1u; }
  double m0, m1, m2;
  hex_m(q, r, m0, m1, m2);
  if (fabs(t0 - p * (m0 - 0.5)) <= kFlagDist || fabs(t0 - p * (m0 + 0.5)) <= kFlagDist ||
      fabs(t1 - p * (m1 - 0.5)) <= kFlagDist || fabs(t1 - p * (m1 + 0.5)) <= kFlagDist ||
      fabs(t2 - p * (m2 - 0.5)) <= kFlagDist || fabs(t2 - p * (m2 + 0.5)) <= kFlagDist)
    flags |= 1u;
  qo = q;
  ro = r;
}


NT_DEV_END
