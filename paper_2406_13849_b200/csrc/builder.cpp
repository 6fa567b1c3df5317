// Host model builder: validation, universe bounding boxes, cell AABBs by truncation,
// per-universe SAH bounding interval hierarchy, optional pseudo-array conversion, and
// flattening into the device tables of nt_layout.hpp.
//
// Paper: CSG cells from surface half-spaces (§1); universes and arrays
// (P:133-145); pseudo-array universes (§4.3 ST method); cell bounding boxes by
// successive truncation; BIH construction with SAH over three equally spaced
// candidate partitions per axis.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <functional>
#include <map>
#include <numeric>

#include "nt_model.hpp"

namespace nt {
namespace {

constexpr double kBig = 1e7;   // finite stand-in for "unbounded" in bounding boxes (cm)

[[noreturn]] void fail(const char* fmt, long a = 0, long b = 0) {
  char buf[256];
  std::snprintf(buf, sizeof buf, fmt, a, b);
  throw GeomError(buf);
}

bool finite(double v) { return std::isfinite(v); }

// ---------------------------------------------------------------- validation
int depth_below(const std::vector<HCell>& C, const std::vector<HUniv>& U, int u,
                std::vector<int>& memo, std::vector<int>& state) {
  if (state[u] == 1) fail("universe cycle through universe %ld", u);
  if (state[u] == 2) return memo[u];
  state[u] = 1;
  int best = 0;
  const HUniv& X = U[u];
  if (X.kind == U_CSG) {
    for (int c : X.cells) {
      int d = C[c].fill_kind == 0 ? 1 : 1 + depth_below(C, U, C[c].fill, memo, state);
      best = std::max(best, d);
    }
  } else {
    for (size_t i = 0; i <= X.fill.size(); ++i) {
      int f = i < X.fill.size() ? X.fill[i] : X.outer;
      if (f < 0) continue;
      best = std::max(best, 1 + depth_below(C, U, f, memo, state));
    }
  }
  state[u] = 2;
  memo[u] = best;
  return best;
}

void validate(const std::vector<HSurf>& S, const std::vector<HMat>& M, const std::vector<HCell>& C,
              const std::vector<HUniv>& U, int root, int& max_depth) {
  const int ns = (int)S.size(), nm = (int)M.size(), nu = (int)U.size();
  if (root < 0 || root >= nu) fail("root universe not set or out of range (%ld)", root);
  for (int i = 0; i < ns; ++i) {
    const HSurf& s = S[i];
    for (double v : s.c) if (!finite(v)) fail("surface %ld has a non-finite coefficient", i);
    if ((s.kind == S_CZ && !(s.c[2] > 0)) || (s.kind == S_SPHERE && !(s.c[3] > 0)))
      fail("surface %ld: radius must be > 0", i);
    if (s.kind == S_PLANE && s.c[0] == 0 && s.c[1] == 0 && s.c[2] == 0)
      fail("surface %ld: zero plane normal", i);
    if (s.bc == 2 && s.kind > S_PZ) fail("surface %ld: REFLECT only on PX/PY/PZ", i);
  }
  for (int i = 0; i < nm; ++i) {
    if (!finite(M[i].st) || !finite(M[i].sa) || M[i].st < 0 || M[i].sa < 0 || M[i].sa > M[i].st)
      fail("material %ld: need 0 <= sigma_a <= sigma_t", i);
    if (!finite(M[i].nusf) || M[i].nusf < 0 || (M[i].nusf > 0 && !(M[i].sa > 0)) || M[i].nusf / (M[i].sa > 0 ? M[i].sa : 1) > 200)
      fail("material %ld: need nu_sigma_f >= 0, sigma_a > 0 when fissile, nu_sigma_f / sigma_a <= 200", i);
  }
  for (int i = 0; i < (int)C.size(); ++i) {
    const HCell& c = C[i];
    std::vector<int> ids = c.sid;
    std::sort(ids.begin(), ids.end());
    for (size_t k = 0; k < ids.size(); ++k) {
      if (ids[k] < 0 || ids[k] >= ns) fail("cell %ld: surface reference out of range", i);
      if (k && ids[k] == ids[k - 1]) fail("cell %ld references surface %ld twice", i, ids[k]);
      if (S[ids[k]].bc != 0 && c.uid != root)
        fail("surface %ld has a boundary condition but is used outside the root universe", ids[k]);
    }
    if (c.fill_kind == 0 && (c.fill < 0 || c.fill >= nm)) fail("cell %ld: bad material", i);
    if (c.fill_kind == 1 && (c.fill < 0 || c.fill >= nu)) fail("cell %ld: bad fill universe", i);
    for (double v : c.tr) if (!finite(v)) fail("cell %ld: non-finite translation", i);
  }
  for (int i = 0; i < nu; ++i) {
    const HUniv& u = U[i];
    if (u.kind == U_RECT && !u.e[0].empty()) {
      for (int a = 0; a < (u.is2d ? 2 : 3); ++a) {
        if ((int)u.e[a].size() != u.n[a] + 1 || u.n[a] < 1) fail("rect array %ld: bad edge count", i);
        for (size_t k = 0; k < u.e[a].size(); ++k)
          if (!finite(u.e[a][k]) || (k && !(u.e[a][k - 1] < u.e[a][k])))
            fail("rect array %ld: edges must be finite and strictly increasing", i);
      }
    } else if (u.kind == U_RECT) {
      if (!(u.p[0] > 0) || !(u.p[1] > 0) || u.p[2] < 0) fail("rect array %ld: bad pitch", i);
      for (int a = 0; a < 3; ++a) {
        if (u.n[a] < 1) fail("rect array %ld: bad shape", i);
        if (!finite(u.ll[a])) fail("rect array %ld: bad lower-left", i);
      }
    } else if (u.kind == U_HEX) {
      if (!(u.pitch > 0) || u.rings < 1 || u.zp < 0 || (u.zp > 0 && u.nz < 1))
        fail("hex array %ld: bad parameters", i);
    }
    if (u.kind != U_CSG) {
      for (int f : u.fill) if (f < 0 || f >= nu) fail("array %ld: bad fill universe", i);
      if (u.outer < -1 || u.outer >= nu) fail("array %ld: bad outer universe", i);
    }
  }
  std::vector<int> memo(nu, 0), state(nu, 0);
  max_depth = depth_below(C, U, root, memo, state);
  if (max_depth > kMaxDepth) fail("nesting depth %ld exceeds %ld", max_depth, kMaxDepth);
  if (max_depth < 1) fail("root universe has no material cells");
}

// ---------------------------------------------------------------- bounding boxes (O23)
Aabb truncate(const std::vector<HSurf>& S, const HCell& c, const Aabb& start) {
  Aabb b = start;
  for (size_t h = 0; h < c.sid.size(); ++h) {
    const HSurf& s = S[c.sid[h]];
    const bool neg = c.sense[h] == 0;
    if (s.kind <= S_PZ) {
      const int a = s.kind;
      if (neg) b.hi[a] = std::min(b.hi[a], s.c[0]);
      else b.lo[a] = std::max(b.lo[a], s.c[0]);
    } else if (s.kind == S_CZ && neg) {
      for (int a = 0; a < 2; ++a) {
        b.lo[a] = std::max(b.lo[a], s.c[a] - s.c[2]);
        b.hi[a] = std::min(b.hi[a], s.c[a] + s.c[2]);
      }
    } else if (s.kind == S_SPHERE && neg) {
      for (int a = 0; a < 3; ++a) {
        b.lo[a] = std::max(b.lo[a], s.c[a] - s.c[3]);
        b.hi[a] = std::min(b.hi[a], s.c[a] + s.c[3]);
      }
    }
  }
  return b;
}

// Tighter box for cells bounded by general planes (e.g. the hexagonal prisms of a pseudo-array
// universe): the box of the polytope {truncated box} ∩ {plane half-spaces}, from its vertices.
// Quadrics are only used through truncate(), so the result still contains the cell.  Falls
// back to the truncated box when the enumeration finds nothing (empty or degenerate cell).
Aabb polytope_box(const std::vector<HSurf>& S, const HCell& c, const Aabb& b, bool empty_if_none = false) {
  struct H { double n[3], d; };             // n.x <= d
  std::vector<H> hs;
  bool general = false;
  for (size_t h = 0; h < c.sid.size(); ++h) {
    const HSurf& s = S[c.sid[h]];
    if (s.kind != S_PLANE) continue;
    general = true;
    const double g = c.sense[h] == 0 ? 1.0 : -1.0;
    hs.push_back({{g * s.c[0], g * s.c[1], g * s.c[2]}, g * s.c[3]});
  }
  if (!general || !b.valid()) return b;
  for (int a = 0; a < 3; ++a) {
    H lo{{0, 0, 0}, -b.lo[a]}, hi{{0, 0, 0}, b.hi[a]};
    lo.n[a] = -1.0;
    hi.n[a] = 1.0;
    hs.push_back(lo);
    hs.push_back(hi);
  }
  double scale = 1.0;
  for (int a = 0; a < 3; ++a) scale = std::max({scale, std::fabs(b.lo[a]), std::fabs(b.hi[a])});
  Aabb r = Aabb::empty();
  const size_t m = hs.size();
  for (size_t i = 0; i < m; ++i)
    for (size_t j = i + 1; j < m; ++j)
      for (size_t k = j + 1; k < m; ++k) {
        const double* A = hs[i].n; const double* B = hs[j].n; const double* C = hs[k].n;
        const double bc[3] = {B[1] * C[2] - B[2] * C[1], B[2] * C[0] - B[0] * C[2], B[0] * C[1] - B[1] * C[0]};
        const double ca[3] = {C[1] * A[2] - C[2] * A[1], C[2] * A[0] - C[0] * A[2], C[0] * A[1] - C[1] * A[0]};
        const double ab[3] = {A[1] * B[2] - A[2] * B[1], A[2] * B[0] - A[0] * B[2], A[0] * B[1] - A[1] * B[0]};
        const double det = A[0] * bc[0] + A[1] * bc[1] + A[2] * bc[2];
        const double na = std::sqrt(A[0] * A[0] + A[1] * A[1] + A[2] * A[2]);
        const double nb = std::sqrt(B[0] * B[0] + B[1] * B[1] + B[2] * B[2]);
        const double nc = std::sqrt(C[0] * C[0] + C[1] * C[1] + C[2] * C[2]);
        if (std::fabs(det) <= 1e-9 * na * nb * nc) continue;
        double p[3];
        for (int a = 0; a < 3; ++a) p[a] = (hs[i].d * bc[a] + hs[j].d * ca[a] + hs[k].d * ab[a]) / det;
        bool in = true;
        for (size_t q = 0; q < m && in; ++q) {
          const double* n = hs[q].n;
          const double nn = std::sqrt(n[0] * n[0] + n[1] * n[1] + n[2] * n[2]);
          in = n[0] * p[0] + n[1] * p[1] + n[2] * p[2] - hs[q].d <= 1e-9 * nn * scale;
        }
        if (in) r.grow(Aabb{{p[0], p[1], p[2]}, {p[0], p[1], p[2]}});
      }
  if (!r.valid()) return empty_if_none ? Aabb::empty() : b;
  for (int a = 0; a < 3; ++a) {          // never looser than the truncated box
    r.lo[a] = std::max(r.lo[a], b.lo[a]);
    r.hi[a] = std::min(r.hi[a], b.hi[a]);
  }
  return r.valid() ? r : b;
}

Aabb shift(const Aabb& b, const double t[3]) {
  Aabb r = b;
  for (int a = 0; a < 3; ++a) { r.lo[a] -= t[a]; r.hi[a] -= t[a]; }
  return r;
}

void topo_order(const std::vector<HCell>& C, const std::vector<HUniv>& U, int u,
                std::vector<int>& seen, std::vector<int>& post) {
  if (seen[u]) return;
  seen[u] = 1;
  const HUniv& X = U[u];
  if (X.kind == U_CSG) {
    for (int c : X.cells) if (C[c].fill_kind == 1) topo_order(C, U, C[c].fill, seen, post);
  } else {
    for (int f : X.fill) topo_order(C, U, f, seen, post);
    if (X.outer >= 0) topo_order(C, U, X.outer, seen, post);
  }
  post.push_back(u);
}

std::vector<Aabb> universe_boxes(const std::vector<HSurf>& S, const std::vector<HCell>& C,
                                 const std::vector<HUniv>& U, int root) {
  std::vector<Aabb> box(U.size(), Aabb::empty());
  std::vector<int> seen(U.size(), 0), post;
  topo_order(C, U, root, seen, post);
  std::reverse(post.begin(), post.end());   // parents before children
  Aabb big{{-kBig, -kBig, -kBig}, {kBig, kBig, kBig}};
  if (U[root].kind == U_CSG) {
    for (int c : U[root].cells) {
      Aabb a = polytope_box(S, C[c], truncate(S, C[c], big));
      if (a.valid()) box[root].grow(a);
    }
  } else {
    box[root] = big;
  }
  for (int u : post) {
    if (!box[u].valid()) continue;
    const HUniv& X = U[u];
    if (X.kind == U_CSG) {
      for (int c : X.cells) {
        if (C[c].fill_kind != 1) continue;
        Aabb a = polytope_box(S, C[c], truncate(S, C[c], box[u]));
        if (a.valid()) box[C[c].fill].grow(shift(a, C[c].tr));
      }
    } else {
      Aabb t;
      if (X.kind == U_RECT && !X.e[0].empty()) {
        // N1: in-lattice daughters see at most half the widest tile; the outer universe fills
        // the half-infinite slabs (handled below)
        for (int a = 0; a < 3; ++a) {
          double w = 0.0;
          if (a < 3 && !X.e[a].empty())
            for (size_t k = 1; k < X.e[a].size(); ++k) w = std::max(w, X.e[a][k] - X.e[a][k - 1]);
          t.lo[a] = -0.5 * w * (1.0 + 1e-9);
          t.hi[a] = 0.5 * w * (1.0 + 1e-9);
        }
        if (X.is2d) { t.lo[2] = box[u].lo[2]; t.hi[2] = box[u].hi[2]; }
        for (int f : X.fill) box[f].grow(t);
        if (X.outer >= 0) box[X.outer].grow(Aabb{{-kBig, -kBig, -kBig}, {kBig, kBig, kBig}});
        continue;
      } else if (X.kind == U_RECT) {
        for (int a = 0; a < 3; ++a) { t.lo[a] = -0.5 * X.p[a]; t.hi[a] = 0.5 * X.p[a]; }
        if (X.is2d) { t.lo[2] = box[u].lo[2]; t.hi[2] = box[u].hi[2]; }
      } else {
        const double rho = X.pitch / std::sqrt(3.0) * (1.0 + 1e-9);
        t.lo[0] = t.lo[1] = -rho;
        t.hi[0] = t.hi[1] = rho;
        if (X.nz > 0) { t.lo[2] = -0.5 * X.zp; t.hi[2] = 0.5 * X.zp; }
        else { t.lo[2] = box[u].lo[2]; t.hi[2] = box[u].hi[2]; }
      }
      for (int f : X.fill) box[f].grow(t);
      if (X.outer >= 0) box[X.outer].grow(t);
    }
  }
  return box;
}

Aabb pad(Aabb b) {
  for (int a = 0; a < 3; ++a) {
    b.lo[a] -= 1e-9 * (1.0 + std::fabs(b.lo[a]));
    b.hi[a] += 1e-9 * (1.0 + std::fabs(b.hi[a]));
  }
  return b;
}

double area(const Aabb& b) {
  double e[3];
  for (int a = 0; a < 3; ++a) e[a] = std::max(0.0, b.hi[a] - b.lo[a]);
  return 2.0 * (e[0] * e[1] + e[1] * e[2] + e[0] * e[2]);
}

// ---------------------------------------------------------------- BIH
struct BihBuilder {
  std::vector<BihNode>& nodes;
  std::vector<int32_t>& leaf;
  const std::vector<Aabb>& cb;   // per global cell (padded)
  int max_leaf;
  double ct, ci;
  int depth = 0;

  // A leaf's cells are tested in order of decreasing box volume: the largest cell (e.g. a pin's
  // moderator, whose box is the whole tile) is the likeliest to hold a query point.  The order only
  // changes how soon the unique containing cell is found (reading O22), never which one.
  void make_leaf(int node, std::vector<int> idx) {
    auto vol = [&](int c) {
      double v = 1.0;
      for (int a = 0; a < 3; ++a) v *= std::max(0.0, cb[c].hi[a] - cb[c].lo[a]);
      return std::isnan(v) ? 0.0 : v;
    };
    std::stable_sort(idx.begin(), idx.end(), [&](int x, int y) { return vol(x) > vol(y); });
    nodes[node].meta = -1 - (int)idx.size();
    nodes[node].a = (int)leaf.size();
    nodes[node].lmax = nodes[node].rmin = 0;
    for (int c : idx) leaf.push_back(c);
  }

  void fill(int node, std::vector<int> idx, int d) {
    depth = std::max(depth, d);
    // depth is bounded by the traversal's register stack (kBihStack); a deeper subtree becomes
    // one larger leaf (still exact: the leaf is scanned linearly)
    if ((int)idx.size() <= max_leaf || d >= kBihStack) { make_leaf(node, idx); return; }
    Aabb nb = Aabb::empty(), cen = Aabb::empty();
    for (int c : idx) {
      nb.grow(cb[c]);
      Aabb p;
      for (int a = 0; a < 3; ++a) p.lo[a] = p.hi[a] = 0.5 * (cb[c].lo[a] + cb[c].hi[a]);
      cen.grow(p);
    }
    auto centre = [&](int c, int a) { return 0.5 * (cb[c].lo[a] + cb[c].hi[a]); };
    const double sa_node = std::max(area(nb), 1e-300);
    double best = 1e308;
    int bax = -1;
    double bpos = 0;
    // SAH: three equally spaced candidate partitions per axis
    for (int a = 0; a < 3; ++a) {
      const double ext = cen.hi[a] - cen.lo[a];
      if (!(ext > 0)) continue;
      for (int k = 1; k <= 3; ++k) {
        const double pos = cen.lo[a] + 0.25 * k * ext;
        Aabb L = Aabb::empty(), R = Aabb::empty();
        int nl = 0, nr = 0;
        for (int c : idx) {
          if (centre(c, a) < pos) { L.grow(cb[c]); ++nl; } else { R.grow(cb[c]); ++nr; }
        }
        if (!nl || !nr) continue;
        const double cost = ct + ci * (area(L) * nl + area(R) * nr) / sa_node;
        if (cost < best) { best = cost; bax = a; bpos = pos; }
      }
    }
    std::vector<int> li, ri;
    if (bax < 0) {   // degenerate: median split on the widest centroid axis
      int a = 0;
      for (int k = 1; k < 3; ++k) if (cen.hi[k] - cen.lo[k] > cen.hi[a] - cen.lo[a]) a = k;
      if (!(cen.hi[a] > cen.lo[a])) { make_leaf(node, idx); return; }
      std::sort(idx.begin(), idx.end(), [&](int x, int y) { return centre(x, a) < centre(y, a); });
      li.assign(idx.begin(), idx.begin() + idx.size() / 2);
      ri.assign(idx.begin() + idx.size() / 2, idx.end());
      bax = a;
    } else {
      for (int c : idx) (centre(c, bax) < bpos ? li : ri).push_back(c);
    }
    double lmax = -1e308, rmin = 1e308;
    for (int c : li) lmax = std::max(lmax, cb[c].hi[bax]);
    for (int c : ri) rmin = std::min(rmin, cb[c].lo[bax]);
    const int a0 = (int)nodes.size();
    nodes.push_back({});
    nodes.push_back({});
    nodes[node].meta = bax;
    nodes[node].a = a0;
    nodes[node].lmax = lmax;
    nodes[node].rmin = rmin;
    fill(a0, li, d + 1);
    fill(a0 + 1, ri, d + 1);
  }
};

// ---------------------------------------------------------------- instances (D1)
// Material-cell instances are numbered by a depth-first enumeration: a CSG universe's cells in
// id order (material cell = 1 instance, fill cell = its universe's instances), an array's tiles
// in fill order, then its outer universe once.  The instance of a walk position is the sum, over
// the levels of its stack, of the instances of the earlier siblings: inst_off[univ_inst[u] + k]
// for child k (CSG: cell position; rect: fill index, outer = n; hex: (kz, r, q) grid position,
// outer = W*W*nz).  inst_mc lists the material-cell bin of every instance (the enumeration).
void build_instance_tables(const std::vector<HCell>& C, const std::vector<HUniv>& U, int root, Flat& F) {
  const int nu = (int)U.size();
  std::vector<int64_t> leaves(nu, -1);
  std::function<int64_t(int)> count = [&](int u) -> int64_t {
    if (leaves[u] >= 0) return leaves[u];
    const HUniv& X = U[u];
    int64_t n = 0;
    if (X.kind == U_CSG) {
      for (int c : X.cells) n += C[c].fill_kind == 0 ? 1 : count(C[c].fill);
    } else {
      for (int f : X.fill) n += count(f);
      if (X.outer >= 0) n += count(X.outer);
    }
    return leaves[u] = std::min<int64_t>(n, int64_t(1) << 40);
  };
  for (int u = 0; u < nu; ++u) count(u);
  F.n_inst = leaves[root];
  if (F.n_inst >= (int64_t(1) << 31)) { F.n_inst = 0; return; }   // too many to index in 32 bits
  F.cell_pos.assign(C.size(), 0);
  F.univ_inst.assign(nu, 0);
  for (int u = 0; u < nu; ++u) {
    const HUniv& X = U[u];
    F.univ_inst[u] = (int32_t)F.inst_off.size();
    int64_t acc = 0;
    if (X.kind == U_CSG) {
      for (size_t k = 0; k < X.cells.size(); ++k) {
        const int c = X.cells[k];
        F.cell_pos[c] = (int32_t)k;
        F.inst_off.push_back((int32_t)acc);
        acc += C[c].fill_kind == 0 ? 1 : leaves[C[c].fill];
      }
    } else if (X.kind == U_RECT) {
      for (int f : X.fill) { F.inst_off.push_back((int32_t)acc); acc += leaves[f]; }
      F.inst_off.push_back((int32_t)acc);                         // outer
    } else {
      const int R = X.rings - 1, W = 2 * R + 1, nzl = X.zp > 0 ? X.nz : 1;
      const int per = (int)X.fill.size() / nzl;
      std::vector<int64_t> prefix(X.fill.size() + 1, 0);
      for (size_t t = 0; t < X.fill.size(); ++t) prefix[t + 1] = prefix[t] + leaves[X.fill[t]];
      std::vector<int32_t> grid((size_t)W * W * nzl + 1, 0);
      for (int kz = 0; kz < nzl; ++kz) {
        int o = 0;
        for (int r = -R; r <= R; ++r)
          for (int q = -R; q <= R; ++q)
            if (std::max({std::abs(q), std::abs(r), std::abs(q + r)}) <= R)
              grid[(size_t)kz * W * W + (r + R) * W + (q + R)] = (int32_t)prefix[(size_t)kz * per + o++];
      }
      grid[(size_t)W * W * nzl] = (int32_t)prefix[X.fill.size()];   // outer
      F.inst_off.insert(F.inst_off.end(), grid.begin(), grid.end());
    }
  }
  // the enumeration itself (material-cell bins are the material cells in global id order)
  std::vector<int32_t> mc_of(C.size(), -1);
  for (int i = 0, k = 0; i < (int)C.size(); ++i) if (C[i].fill_kind == 0) mc_of[i] = k++;
  F.inst_mc.clear();
  F.inst_mc.reserve((size_t)F.n_inst);
  std::function<void(int)> walk = [&](int u) {
    const HUniv& X = U[u];
    if (X.kind == U_CSG) {
      for (int c : X.cells) {
        if (C[c].fill_kind == 0) F.inst_mc.push_back(mc_of[c]);
        else walk(C[c].fill);
      }
    } else {
      for (int f : X.fill) walk(f);
      if (X.outer >= 0) walk(X.outer);
    }
  };
  walk(root);
}

// ---------------------------------------------------------------- pseudo-arrays
// Replace every rect/hex array universe by a CSG universe of explicit tile cells (same uid,
// same depth), covering the in-lattice tiles and every out-of-lattice tile that meets the
// universe bounding box; out-of-lattice tiles take `outer` (skipped when there is none).
void convert_pseudo_arrays(std::vector<HSurf>& S, std::vector<HCell>& C, std::vector<HUniv>& U,
                           const std::vector<Aabb>& box) {
  for (int u = 0; u < (int)U.size(); ++u) {
    HUniv& X = U[u];
    if (X.kind == U_CSG || !box[u].valid()) continue;
    if (X.kind == U_RECT && !X.e[0].empty()) {
      // N1: every tile -1..n per axis; the slabs -1 / n are bounded on one side only
      const int na = X.is2d ? 2 : 3;
      std::vector<int> plane[3];
      for (int a = 0; a < na; ++a)
        for (double v : X.e[a]) {
          plane[a].push_back((int)S.size());
          S.push_back(HSurf{a, 0, {v, 0, 0, 0}});
        }
      HUniv Y;
      Y.kind = U_CSG;
      const int hk = na == 3 ? X.n[2] : 0, lk = na == 3 ? -1 : 0;
      for (int k = lk; k <= hk; ++k)
        for (int j = -1; j <= X.n[1]; ++j)
          for (int i = -1; i <= X.n[0]; ++i) {
            const int ijk[3] = {i, j, k};
            bool in = true;
            for (int a = 0; a < na; ++a) in = in && ijk[a] >= 0 && ijk[a] < X.n[a];
            const int d = in ? X.fill[i + X.n[0] * (j + X.n[1] * (na == 3 ? k : 0))] : X.outer;
            if (d < 0) continue;
            HCell c;
            c.uid = u;
            c.fill_kind = 1;
            c.fill = d;
            for (int a = 0; a < 3; ++a) {
              if (a >= na) { c.tr[a] = 0.0; continue; }
              const int n = X.n[a], t = ijk[a];
              c.tr[a] = t < 0 ? X.e[a][0] : t >= n ? X.e[a][n] : (X.e[a][t] + X.e[a][t + 1]) * 0.5;
            }
            for (int a = 0; a < na; ++a) {
              if (ijk[a] >= 0) { c.sid.push_back(plane[a][ijk[a]]); c.sense.push_back(1); }
              if (ijk[a] < X.n[a]) { c.sid.push_back(plane[a][ijk[a] + 1]); c.sense.push_back(0); }
            }
            Y.cells.push_back((int)C.size());
            C.push_back(c);
          }
      X = Y;
    } else if (X.kind == U_RECT) {
      const int na = X.is2d ? 2 : 3;
      int lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
      std::vector<int> plane0[3];
      for (int a = 0; a < na; ++a) {
        lo[a] = std::min(0, (int)std::floor((box[u].lo[a] - X.ll[a]) / X.p[a]) - 1);
        hi[a] = std::max(X.n[a] - 1, (int)std::floor((box[u].hi[a] - X.ll[a]) / X.p[a]) + 1);
        for (int i = lo[a]; i <= hi[a] + 1; ++i) {   // e(i) = LL + i p  (O8: mul then add)
          HSurf s{a, 0, {X.ll[a] + (double)i * X.p[a], 0, 0, 0}};
          plane0[a].push_back((int)S.size());
          S.push_back(s);
        }
      }
      HUniv Y;
      Y.kind = U_CSG;
      for (int k = lo[2]; k <= hi[2]; ++k)
        for (int j = lo[1]; j <= hi[1]; ++j)
          for (int i = lo[0]; i <= hi[0]; ++i) {
            const int ijk[3] = {i, j, k};
            bool in = true;
            for (int a = 0; a < na; ++a) in = in && ijk[a] >= 0 && ijk[a] < X.n[a];
            const int d = in ? X.fill[i + X.n[0] * (j + X.n[1] * (na == 3 ? k : 0))] : X.outer;
            if (d < 0) continue;
            HCell c;
            c.uid = u;
            c.fill_kind = 1;
            c.fill = d;
            for (int a = 0; a < 3; ++a)
              c.tr[a] = a < na ? X.ll[a] + ((double)ijk[a] + 0.5) * X.p[a] : 0.0;
            for (int a = 0; a < na; ++a) {
              c.sid.push_back(plane0[a][ijk[a] - lo[a]]);
              c.sense.push_back(1);
              c.sid.push_back(plane0[a][ijk[a] - lo[a] + 1]);
              c.sense.push_back(0);
            }
            Y.cells.push_back((int)C.size());
            C.push_back(c);
          }
      X = Y;
    } else {   // HEX: tile (q,r) = intersection over k of m_k - 1/2 <= t_k < m_k + 1/2 (O9)
      const double H = kHexH, p = X.pitch, pH = p * H;
      double n[3][2];
      if (X.orient == 0) { double v[3][2] = {{1.0, 0.0}, {0.5, H}, {-0.5, H}}; std::copy(&v[0][0], &v[0][0] + 6, &n[0][0]); }
      else { double v[3][2] = {{H, 0.5}, {0.0, 1.0}, {-H, 0.5}}; std::copy(&v[0][0], &v[0][0] + 6, &n[0][0]); }
      double a1[2], a2[2];
      if (X.orient == 0) { a1[0] = p; a1[1] = 0.0; a2[0] = p * 0.5; a2[1] = pH; }
      else { a1[0] = pH; a1[1] = p * 0.5; a2[0] = 0.0; a2[1] = p; }
      const int R = X.rings - 1;
      const double reach = std::max({std::fabs(box[u].lo[0] - X.C[0]), std::fabs(box[u].hi[0] - X.C[0]),
                                     std::fabs(box[u].lo[1] - X.C[1]), std::fabs(box[u].hi[1] - X.C[1])});
      const int W = std::max(R, (int)std::ceil(reach / (0.5 * p)) + 2);
      // collect tiles whose hexagon meets the box (centre within box + circumradius)
      const double rho = p / std::sqrt(3.0) + 1e-9;
      std::vector<std::array<int, 2>> tiles;
      for (int r = -W; r <= W; ++r)
        for (int q = -W; q <= W; ++q) {
          const double cx = X.C[0] + ((double)q * a1[0] + (double)r * a2[0]);
          const double cy = X.C[1] + ((double)q * a1[1] + (double)r * a2[1]);
          const bool inl = std::max({std::abs(q), std::abs(r), std::abs(q + r)}) <= R;
          if (inl || (cx + rho >= box[u].lo[0] && cx - rho <= box[u].hi[0] && cy + rho >= box[u].lo[1] &&
                      cy - rho <= box[u].hi[1]))
            tiles.push_back({q, r});
        }
      // planes n_k . x = n_k . C + p * b for half-integer b (2b integer key), family order
      std::map<std::pair<int, int>, int> plane;
      auto m_of = [](int q, int r, int k) {
        return k == 0 ? (double)q + (double)r * 0.5
                      : (k == 1 ? (double)q * 0.5 + (double)r : -((double)q * 0.5) + (double)r * 0.5);
      };
      for (int k = 0; k < 3; ++k) {
        std::vector<int> keys;
        for (auto& t : tiles) {
          const double m = m_of(t[0], t[1], k);
          keys.push_back((int)std::lround(2.0 * (m - 0.5)));
          keys.push_back((int)std::lround(2.0 * (m + 0.5)));
        }
        std::sort(keys.begin(), keys.end());
        keys.erase(std::unique(keys.begin(), keys.end()), keys.end());
        for (int key : keys) {
          HSurf s{S_PLANE, 0, {n[k][0], n[k][1], 0.0,
                               (n[k][0] * X.C[0] + n[k][1] * X.C[1]) + p * (0.5 * key)}};
          plane[{k, key}] = (int)S.size();
          S.push_back(s);
        }
      }
      const int nzl = X.nz > 0 ? X.nz : 1;
      int klo = 0, khi = 0;
      std::vector<int> zpl;
      if (X.nz > 0) {
        klo = std::min(0, (int)std::floor((box[u].lo[2] - X.zlo) / X.zp) - 1);
        khi = std::max(X.nz - 1, (int)std::floor((box[u].hi[2] - X.zlo) / X.zp) + 1);
        for (int k = klo; k <= khi + 1; ++k) {
          HSurf s{S_PZ, 0, {X.zlo + (double)k * X.zp, 0, 0, 0}};
          zpl.push_back((int)S.size());
          S.push_back(s);
        }
      }
      // O9 fill index of in-lattice tiles
      std::map<std::pair<int, int>, int> order;
      int cnt = 0;
      for (int r = -R; r <= R; ++r)
        for (int q = -R; q <= R; ++q)
          if (std::max({std::abs(q), std::abs(r), std::abs(q + r)}) <= R) order[{q, r}] = cnt++;
      HUniv Y;
      Y.kind = U_CSG;
      for (int kz = klo; kz <= khi; ++kz)
        for (auto& t : tiles) {
          const int q = t[0], r = t[1];
          auto it = order.find({q, r});
          const bool in = it != order.end() && (X.nz == 0 || (kz >= 0 && kz < X.nz));
          const int d = in ? X.fill[it->second + (X.nz > 0 ? kz * (int)(X.fill.size() / nzl) : 0)] : X.outer;
          if (d < 0) continue;
          HCell c;
          c.uid = u;
          c.fill_kind = 1;
          c.fill = d;
          c.tr[0] = X.C[0] + ((double)q * a1[0] + (double)r * a2[0]);
          c.tr[1] = X.C[1] + ((double)q * a1[1] + (double)r * a2[1]);
          c.tr[2] = X.nz > 0 ? X.zlo + ((double)kz + 0.5) * X.zp : 0.0;
          for (int k = 0; k < 3; ++k) {
            const double m = m_of(q, r, k);
            c.sid.push_back(plane[{k, (int)std::lround(2.0 * (m - 0.5))}]);
            c.sense.push_back(1);
            c.sid.push_back(plane[{k, (int)std::lround(2.0 * (m + 0.5))}]);
            c.sense.push_back(0);
          }
          if (X.nz > 0) {
            c.sid.push_back(zpl[kz - klo]);
            c.sense.push_back(1);
            c.sid.push_back(zpl[kz - klo + 1]);
            c.sense.push_back(0);
          }
          Y.cells.push_back((int)C.size());
          C.push_back(c);
        }
      X = Y;
    }
  }
}

double surf_tol(const HSurf& s) {   // O16: 1e-10 x |grad f| scale (same formula as documented)
  if (s.kind == S_CZ) return kFlagDist * (2.0 * s.c[2]);
  if (s.kind == S_SPHERE) return kFlagDist * (2.0 * s.c[3]);
  if (s.kind == S_PLANE) return kFlagDist * std::sqrt((s.c[0] * s.c[0] + s.c[1] * s.c[1]) + s.c[2] * s.c[2]);
  return kFlagDist;
}

}  // namespace

void build_rect_tables(const std::vector<HSurf>& S, const std::vector<HMat>& M,
                       const std::vector<HCell>& C, const std::vector<HUniv>& U, int root,
                       Flat& F);   // rect_spec.cpp

void build_flat(const std::vector<HSurf>& s_in, const std::vector<HMat>& M,
                const std::vector<HCell>& c_in, const std::vector<HUniv>& u_in, int root,
                const BuildOpts& opts, Flat& F) {
  F = Flat();
  int depth = 0;
  validate(s_in, M, c_in, u_in, root, depth);
  std::vector<HSurf> S = s_in;
  std::vector<HCell> C = c_in;
  std::vector<HUniv> U = u_in;
  std::vector<Aabb> ubox = universe_boxes(S, C, U, root);
  if (opts.pseudo) {
    convert_pseudo_arrays(S, C, U, ubox);
    ubox = universe_boxes(S, C, U, root);
  } else {
    build_rect_tables(S, M, C, U, root, F);
  }
  F.root = root;
  F.max_depth = depth;

  // feature set of the (converted) model: selects the compiled kernel variant
  for (const HSurf& s : S) {
    if (s.kind == S_PLANE) F.features |= F_PLANE;
    if (s.kind == S_SPHERE) F.features |= F_SPHERE;
  }
  for (const HUniv& u : U) {
    if (u.kind == U_HEX) F.features |= F_HEX;
    if (u.kind == U_RECT && !u.e[0].empty()) F.features |= F_RECTNU;
  }
  // surfaces
  for (const HSurf& s : S) {
    DSurf d{};
    if (s.kind <= S_PZ) d.c[0] = s.c[0];
    else if (s.kind == S_PLANE) for (int k = 0; k < 4; ++k) d.c[k] = s.c[k];
    else if (s.kind == S_CZ) { d.c[0] = s.c[0]; d.c[1] = s.c[1]; d.c[2] = s.c[2] * s.c[2]; }
    else { d.c[0] = s.c[0]; d.c[1] = s.c[1]; d.c[2] = s.c[2]; d.c[3] = s.c[3] * s.c[3]; }
    F.surf.push_back(d);
    F.surf_tol.push_back(surf_tol(s));
    F.surf_meta.push_back((uint8_t)(s.kind | (s.bc << 4)));
  }
  // cells: half-spaces sorted by surface id (O13), material-cell bins in cell-id order (O20)
  F.cell_hs.push_back(0);
  for (int i = 0; i < (int)C.size(); ++i) {
    const HCell& c = C[i];
    std::vector<int> o(c.sid.size());
    std::iota(o.begin(), o.end(), 0);
    std::sort(o.begin(), o.end(), [&](int a, int b) { return c.sid[a] < c.sid[b]; });
    for (int k : o) {
      F.hs.push_back(hs_pack(c.sid[k], S[c.sid[k]].kind, c.sense[k]));
      DHs r{};
      for (int q = 0; q < 4; ++q) r.c[q] = F.surf[c.sid[k]].c[q];
      // CZ: c3 (unused by f and the distance) carries R for the safety bound |rho - R|
      if (S[c.sid[k]].kind == S_CZ) r.c[3] = std::sqrt(r.c[2]);
      r.e = F.hs.back();
      r.meta = F.surf_meta[c.sid[k]];
      r.tol = F.surf_tol[c.sid[k]];
      F.hsr.push_back(r);
    }
    // slab pairs: two consecutive half-spaces of the same axis plane kind with opposite senses (a cell
    // between two PX / PY / PZ planes).  Only the one the flight heads towards can be exited, so the
    // distance loop evaluates the pair with one division (kHsSlab on the first entry)
    for (size_t k = F.cell_hs.back(); k + 1 < F.hsr.size(); ++k) {
      const int e0 = F.hsr[k].e, e1 = F.hsr[k + 1].e;
      if (hs_kind(e0) <= S_PZ && hs_kind(e1) == hs_kind(e0) && hs_sense(e0) != hs_sense(e1)) {
        F.hsr[k].meta |= kHsSlab;
        ++k;
      }
    }
    F.cell_hs.push_back((int32_t)F.hs.size());
    if (c.fill_kind == 0) {
      F.cell_fill.push_back(F.n_mc++);
      const HMat& m = M[c.fill];
      F.mc_st.push_back(m.st);
      F.mc_pabs.push_back(m.st > 0.0 ? m.sa / m.st : 0.0);
      const double nut = m.nusf > 0.0 ? m.nusf / m.sa : 0.0;      // F1: IEEE division, once
      F.mc_nut.push_back(nut);
      F.max_sites = std::max(F.max_sites, (int)std::floor(nut) + 1);
      F.mc_cell.push_back(i);
    } else {
      F.cell_fill.push_back(-1 - c.fill);
    }
    for (int a = 0; a < 3; ++a) F.cell_tr.push_back(c.tr[a]);
  }
  // Across-surface neighbours, a search shortcut for CSG crossings (Alg. 8): for half-space entry h
  // of cell c (surface s, sense t), the cells of c's universe that hold s with the other sense.
  // Lists longer than kNbMax stay empty (the BIH search is used); the containing cell is unique,
  // so testing these first changes nothing but the search time.
  {
    constexpr int kNbMax = 4;
    F.hs_nb_off.assign(1, 0);
    F.nb_cells.clear();
    std::map<std::pair<int, int>, std::vector<int>> by_side;    // (surface, sense) -> cells, per universe
    std::vector<int> uni_of(C.size(), -1);
    for (int u = 0; u < (int)U.size(); ++u)
      if (U[u].kind == U_CSG) for (int c : U[u].cells) uni_of[c] = u;
    std::vector<std::map<std::pair<int, int>, std::vector<int>>> side(U.size());
    for (int i = 0; i < (int)C.size(); ++i)
      if (uni_of[i] >= 0)
        for (size_t k = 0; k < C[i].sid.size(); ++k) side[uni_of[i]][{C[i].sid[k], C[i].sense[k]}].push_back(i);
    for (int i = 0; i < (int)C.size(); ++i) {
      for (int h = F.cell_hs[i]; h < F.cell_hs[i + 1]; ++h) {
        const int e = F.hs[h], s = e >> 4, t = e & 1;
        if (uni_of[i] >= 0) {
          auto it = side[uni_of[i]].find({s, t ^ 1});
          if (it != side[uni_of[i]].end() && (int)it->second.size() <= kNbMax)
            for (int c2 : it->second) F.nb_cells.push_back(c2);
        }
        F.hs_nb_off.push_back((int32_t)F.nb_cells.size());
      }
    }
    if (F.nb_cells.empty()) F.nb_cells.push_back(0);
  }
  // cell AABBs by truncation of the universe box, padded
  std::vector<Aabb> cb(C.size(), Aabb::empty());
  for (int u = 0; u < (int)U.size(); ++u)
    if (U[u].kind == U_CSG)
      for (int c : U[u].cells) {
        // empty_if_none: a plane-bounded cell whose polytope misses the universe box is detected
        // here and gets its own (natural) box below, which always contains the cell
        Aabb a = ubox[u].valid() ? polytope_box(S, C[c], truncate(S, C[c], ubox[u]), true)
                                 : Aabb{{-kBig, -kBig, -kBig}, {kBig, kBig, kBig}};
        if (!a.valid()) {
          // the cell does not meet the universe box (e.g. pseudo-array tiles beyond it): no point
          // the walk can reach lies in it.  Give it its own box outside, so that the BIH keeps it
          // away from every query (a universe-sized box would put it in every search).
          const Aabb big{{-kBig, -kBig, -kBig}, {kBig, kBig, kBig}};
          a = polytope_box(S, C[c], truncate(S, C[c], big));
          if (!a.valid()) a = ubox[u].valid() ? ubox[u] : Aabb{{0, 0, 0}, {0, 0, 0}};
        }
        cb[c] = pad(a);
      }
  if (!opts.pseudo) build_instance_tables(C, U, root, F);
  // universes
  F.bih_depth.assign(U.size(), 0);
  for (int u = 0; u < (int)U.size(); ++u) {
    const HUniv& X = U[u];
    DUniv d{};
    d.kind = X.kind;
    d.outer = X.outer;
    d.fill_off = (int32_t)F.fills.size();
    if (X.kind == U_CSG) {
      BihBuilder B{F.bih, F.bih_leaf, cb, std::max(1, opts.max_leaf), opts.ct, opts.ci};
      const int node = (int)F.bih.size();
      F.bih.push_back({});
      B.fill(node, X.cells, 0);
      F.bih_depth[u] = B.depth;
      if ((int)F.bih.size() - node >= 65535) fail("BIH of universe %ld has more than 65535 nodes", u);
      d.i0 = node;
      d.i1 = X.cells.empty() ? 0 : X.cells.front();
      d.i2 = (int)X.cells.size();
    } else if (X.kind == U_RECT) {
      d.i0 = X.n[0]; d.i1 = X.n[1]; d.i2 = X.is2d ? 1 : X.n[2];
      d.is2d = X.is2d;
      for (int a = 0; a < 3; ++a) { d.d[a] = X.ll[a]; d.d[3 + a] = X.p[a]; }
      d.ntile = -1;
      if (!X.e[0].empty()) {                       // N1 edge table: x, y, z (z only in 3-D)
        d.ntile = (int32_t)F.edges.size();
        for (int a = 0; a < (X.is2d ? 2 : 3); ++a) F.edges.insert(F.edges.end(), X.e[a].begin(), X.e[a].end());
      }
      for (int f : X.fill) F.fills.push_back(f);
    } else {
      const double H = kHexH, p = X.pitch;
      const int R = X.rings - 1, W = 2 * R + 1;
      d.i0 = R; d.i1 = X.zp > 0 ? X.nz : 0; d.i2 = X.orient;
      d.ntile = W * W;
      d.d[0] = X.C[0]; d.d[1] = X.C[1]; d.d[2] = p; d.d[3] = p * H;
      d.d[4] = X.zlo; d.d[5] = X.zp;
      if (X.orient == 0) {
        d.d[6] = p; d.d[7] = 0.0; d.d[8] = p * 0.5; d.d[9] = d.d[3];
        const double nv[6] = {1.0, 0.0, 0.5, H, -0.5, H};
        for (int k = 0; k < 6; ++k) d.d[10 + k] = nv[k];
      } else {
        d.d[6] = d.d[3]; d.d[7] = p * 0.5; d.d[8] = 0.0; d.d[9] = p;
        const double nv[6] = {H, 0.5, 0.0, 1.0, -H, 0.5};
        for (int k = 0; k < 6; ++k) d.d[10 + k] = nv[k];
      }
      const int nzl = d.i1 > 0 ? d.i1 : 1;
      const int per = (int)X.fill.size() / nzl;
      std::vector<int32_t> map(W * W, -1);
      int cnt = 0;
      for (int r = -R; r <= R; ++r)
        for (int q = -R; q <= R; ++q)
          if (std::max({std::abs(q), std::abs(r), std::abs(q + r)}) <= R) map[(r + R) * W + (q + R)] = cnt++;
      if (cnt != per) fail("hex array %ld: fill has the wrong length", u);
      for (int kz = 0; kz < nzl; ++kz)
        for (int e = 0; e < W * W; ++e) F.fills.push_back(map[e] < 0 ? -1 : X.fill[kz * per + map[e]]);
    }
    F.univ.push_back(d);
  }
  if (F.bih.empty()) F.bih.push_back({});
  if (F.bih_leaf.empty()) F.bih_leaf.push_back(0);
  if (F.fills.empty()) F.fills.push_back(-1);
  if (F.edges.empty()) F.edges.push_back(0.0);
  if (F.univ_inst.empty()) F.univ_inst.push_back(0);
  if (F.inst_off.empty()) F.inst_off.push_back(0);
  if (F.cell_pos.empty()) F.cell_pos.push_back(0);
  if (F.hs.empty()) F.hs.push_back(0);
  if (F.hsr.empty()) F.hsr.push_back(DHs{});
  if (F.mc_st.empty()) fail("model has no material cells");
}

}  // namespace nt
