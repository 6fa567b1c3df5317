// Rect-specialised tracker tables and gating (§3.3, Alg. 9-10): the model
// must be "root (axis box, or concentric CZ annuli between a PZ pair) -> K rect arrays ->
// concentric-CZ pin", every level holding one universe kind.  The RECT tracker then unrolls the
// K + 2 levels at compile time and uses non-polymorphic per-level code.  If any condition
// fails, rect_ok = false and nt_track(NT_TRACKER_RECT) returns NT_E_UNSUPPORTED with the reason.
#include <algorithm>
#include <cmath>
#include <numeric>
#include <set>

#include "nt_model.hpp"

namespace nt {
namespace {

struct Reject { std::string why; };

std::vector<std::pair<int, int>> sorted_hs(const HCell& c) {
  std::vector<std::pair<int, int>> v;
  for (size_t i = 0; i < c.sid.size(); ++i) v.push_back({c.sid[i], c.sense[i]});
  std::sort(v.begin(), v.end());
  return v;
}

}  // namespace

void build_rect_tables(const std::vector<HSurf>& S, const std::vector<HMat>& M, const std::vector<HCell>& C,
                       const std::vector<HUniv>& U, int root, Flat& F) {
  (void)M;
  F.rect_ok = false;
  RectGeom& rg = F.rg;
  rg = RectGeom{};
  // material-cell index of each cell (same numbering as the flat tables: cell-id order)
  std::vector<int> mc_of(C.size(), -1);
  for (int i = 0, n = 0; i < (int)C.size(); ++i) if (C[i].fill_kind == 0) mc_of[i] = n++;
  try {
    const HUniv& R = U[root];
    if (R.kind != U_CSG) throw Reject{"root universe is not CSG"};
    int child = -1;
    if (R.cells.size() == 1) {   // axis box root
      const HCell& c = C[R.cells[0]];
      auto hs = sorted_hs(c);
      if (hs.size() != 6 || c.fill_kind != 1) throw Reject{"root box cell must have 6 planes and a fill"};
      static const int kind[6] = {S_PX, S_PX, S_PY, S_PY, S_PZ, S_PZ}, sense[6] = {1, 0, 1, 0, 1, 0};
      for (int k = 0; k < 6; ++k) {
        if (S[hs[k].first].kind != kind[k] || hs[k].second != sense[k])
          throw Reject{"root box planes not in canonical id order PX-,PX+,PY-,PY+,PZ-,PZ+"};
        rg.box_sid[k] = hs[k].first;
      }
      rg.root_box = 1;
      rg.root_fill_cell = R.cells[0];
      child = c.fill;
    } else {                     // concentric CZ annuli between one PZ pair
      int zlo = -1, zhi = -1;
      struct Ann { double r2; int cell; int inner_sid, outer_sid; };
      std::vector<Ann> ann;
      double x0 = 0, y0 = 0;
      bool first = true;
      for (int cid : R.cells) {
        const HCell& c = C[cid];
        Ann a{0, cid, -1, -1};
        int nz = 0;
        for (auto [sid, sense] : sorted_hs(c)) {
          const HSurf& s = S[sid];
          if (s.kind == S_PZ) {
            int& slot = sense ? zlo : zhi;
            if (slot >= 0 && slot != sid) throw Reject{"root cells use different PZ planes"};
            slot = sid;
            ++nz;
          } else if (s.kind == S_CZ) {
            if (first) { x0 = s.c[0]; y0 = s.c[1]; first = false; }
            if (s.c[0] != x0 || s.c[1] != y0) throw Reject{"root cylinders are not concentric"};
            if (sense) { if (a.inner_sid >= 0) throw Reject{"root cell with two inner cylinders"}; a.inner_sid = sid; }
            else { if (a.outer_sid >= 0) throw Reject{"root cell with two outer cylinders"}; a.outer_sid = sid; }
          } else {
            throw Reject{"root cell uses a surface other than PZ / CZ"};
          }
        }
        if (nz != 2 || a.outer_sid < 0) throw Reject{"root annulus must be bounded by a PZ pair and an outer CZ"};
        a.r2 = S[a.outer_sid].c[2];
        ann.push_back(a);
      }
      std::sort(ann.begin(), ann.end(), [](const Ann& p, const Ann& q) { return p.r2 < q.r2; });
      if (ann.size() > 16) throw Reject{"more than 16 root annuli"};
      if (zlo < 0 || zhi < 0 || zlo > zhi) throw Reject{"root PZ pair must be (lower, upper) in id order"};
      for (size_t k = 0; k < ann.size(); ++k) {
        const int want_inner = k ? ann[k - 1].outer_sid : -1;
        if (ann[k].inner_sid != want_inner) throw Reject{"root annuli are not nested"};
        if (k && !(ann[k].outer_sid > ann[k - 1].outer_sid)) throw Reject{"root cylinder ids not ascending"};
        if (ann[k].outer_sid < zhi) throw Reject{"root PZ ids must precede the cylinder ids"};
        const HCell& c = C[ann[k].cell];
        if (k == 0) {
          if (c.fill_kind != 1) throw Reject{"innermost root annulus must hold the core array"};
          child = c.fill;
          rg.root_fill_cell = ann[k].cell;
        } else if (c.fill_kind != 0) {
          throw Reject{"outer root annuli must be material cells"};
        }
        rg.root_sid[k] = ann[k].outer_sid;
        rg.root_cell[k] = ann[k].cell;
        rg.root_mc[k] = mc_of[ann[k].cell];
      }
      rg.root_box = 0;
      rg.n_root_cells = (int)ann.size();
      rg.zsid[0] = zlo;
      rg.zsid[1] = zhi;
    }
    // level chain: K rect levels, then pins
    std::set<int> level{child};
    int K = 0;
    for (;;) {
      bool all_rect = true, all_csg = true;
      for (int u : level) { all_rect &= U[u].kind == U_RECT; all_csg &= U[u].kind == U_CSG; }
      if (all_csg) break;
      if (!all_rect) throw Reject{"a level mixes universe kinds (or holds a hex array)"};
      for (int u : level)
        if (!U[u].e[0].empty()) throw Reject{"non-uniform rect array (binary-search lattice)"};
      if (++K > 4) throw Reject{"more than 4 rect levels"};
      std::set<int> next;
      for (int u : level) {
        for (int f : U[u].fill) next.insert(f);
        if (U[u].outer >= 0) next.insert(U[u].outer);
      }
      level = next;
    }
    // pins: concentric CZs about the tile centre, ids ascending with radius, material fills
    F.r_pin_of_univ.assign(U.size(), -1);
    F.r_pin_off.assign(1, 0);
    F.r_pin_sid.clear(); F.r_pin_mc.clear();
    int np = 0;
    for (int u : level) {
      const HUniv& P = U[u];
      struct Ann { double r2; int cell, inner, outer; };
      std::vector<Ann> ann;
      for (int cid : P.cells) {
        const HCell& c = C[cid];
        if (c.fill_kind != 0) throw Reject{"pin cells must be material cells"};
        Ann a{1e300, cid, -1, -1};
        for (auto [sid, sense] : sorted_hs(c)) {
          const HSurf& s = S[sid];
          if (s.kind != S_CZ || s.c[0] != 0.0 || s.c[1] != 0.0) throw Reject{"pin surfaces must be centred CZs"};
          if (sense) { if (a.inner >= 0) throw Reject{"pin cell with two inner cylinders"}; a.inner = sid; }
          else { if (a.outer >= 0) throw Reject{"pin cell with two outer cylinders"}; a.outer = sid; }
        }
        if (a.outer >= 0) a.r2 = S[a.outer].c[2];
        ann.push_back(a);
      }
      std::sort(ann.begin(), ann.end(), [](const Ann& p, const Ann& q) { return p.r2 < q.r2; });
      for (size_t k = 0; k < ann.size(); ++k) {
        const int want_inner = k ? ann[k - 1].outer : -1;
        if (ann[k].inner != want_inner || (k + 1 < ann.size()) != (ann[k].outer >= 0))
          throw Reject{"pin annuli are not nested"};
        if (k && k + 1 < ann.size() && !(ann[k].outer > ann[k - 1].outer)) throw Reject{"pin cylinder ids not ascending"};
        if (k + 1 < ann.size()) F.r_pin_sid.push_back(ann[k].outer);
        F.r_pin_mc.push_back(mc_of[ann[k].cell]);
      }
      F.r_pin_of_univ[u] = np++;
      F.r_pin_off.push_back((int)F.r_pin_sid.size());
    }
    // pin_mc is laid out with (ncz + 1) entries per pin: offset = pin_off[p] + p
    rg.K = K;
    rg.root_univ_child = child;
    F.rect_K = K;
    F.rect_ok = true;
    F.rect_why.clear();
  } catch (const Reject& r) {
    F.rect_ok = false;
    F.rect_why = r.why;
  }
  // keep the device blob non-empty
  auto nz = [](auto& v) { if (v.empty()) v.push_back({}); };
  nz(F.r_pin_of_univ); nz(F.r_pin_off); nz(F.r_pin_sid); nz(F.r_pin_mc);
}

}  // namespace nt
