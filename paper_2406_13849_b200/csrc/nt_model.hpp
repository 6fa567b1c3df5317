// Host-side model (builder input) and the flattened tables produced by nt_finalize.
#pragma once
#include <array>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "nt_layout.hpp"

namespace nt {

struct HSurf { int kind, bc; double c[4]; };
struct HMat { double st, sa, nusf = 0.0; };
struct HCell {
  int uid;
  std::vector<int> sid, sense;   // as given; sorted during flattening
  int fill_kind, fill;           // 0 material, 1 universe
  double tr[3];
};
struct HUniv {
  int kind;                      // U_CSG / U_RECT / U_HEX
  std::vector<int> cells;        // CSG
  double ll[3] = {0, 0, 0}, p[3] = {0, 0, 0};
  int n[3] = {1, 1, 1};
  bool is2d = false;
  int orient = 0, rings = 1, nz = 0;
  double C[2] = {0, 0}, pitch = 0, zlo = 0, zp = 0;
  std::vector<double> e[3];      // non-uniform rect (N1): increasing edges per axis (empty: uniform)
  std::vector<int> fill;         // rect: x fastest; hex: O9 order (x nz layers)
  int outer = -1;
};

struct Aabb {
  double lo[3], hi[3];
  static Aabb empty() { return {{1e300, 1e300, 1e300}, {-1e300, -1e300, -1e300}}; }
  bool valid() const { return lo[0] <= hi[0] && lo[1] <= hi[1] && lo[2] <= hi[2]; }
  void grow(const Aabb& b) {
    for (int a = 0; a < 3; ++a) {
      if (b.lo[a] < lo[a]) lo[a] = b.lo[a];
      if (b.hi[a] > hi[a]) hi[a] = b.hi[a];
    }
  }
};

struct GeomError : std::runtime_error { using std::runtime_error::runtime_error; };

// Flattened host copy of the device blob (see nt_layout.hpp).
struct Flat {
  std::vector<DSurf> surf;
  std::vector<double> surf_tol;
  std::vector<uint8_t> surf_meta;
  std::vector<int32_t> hs, cell_hs, cell_fill;
  std::vector<DHs> hsr;             // hs[h] with its surface's coefficients and tolerance
  std::vector<double> cell_tr;
  std::vector<DUniv> univ;
  std::vector<BihNode> bih;
  std::vector<int32_t> bih_leaf, fills;
  std::vector<double> mc_st, mc_pabs, mc_nut;   // mc_nut: nu Sigma_f / Sigma_a (F1)
  int max_sites = 1;                           // F1: floor(max nut) + 1
  std::vector<int32_t> mc_cell;
  std::vector<double> edges;        // non-uniform rect edges (N1)
  // per-instance tallies (D1): instance = sum over levels of inst_off[univ_inst[u] + child]
  std::vector<int32_t> univ_inst, inst_off, cell_pos, inst_mc;
  std::vector<int32_t> hs_nb_off, nb_cells;   // across-surface neighbours per half-space entry
  int64_t n_inst = 0;               // 0: not available (pseudo-array builds)
  std::vector<int32_t> bih_depth;   // per universe (CSG), host info
  int root = -1, max_depth = 0, n_mc = 0, features = 0;
  // rect-specialised tables
  bool rect_ok = false;
  int rect_K = 0;
  std::string rect_why;
  RectGeom rg{};
  std::vector<int32_t> r_pin_of_univ, r_pin_off, r_pin_sid, r_pin_mc;
};

struct BuildOpts { int device = 0, max_leaf = 4, pseudo = 0; double ct = 1.0, ci = 1.0; };

// builder.cpp
void build_flat(const std::vector<HSurf>& s_in, const std::vector<HMat>& mats,
                const std::vector<HCell>& c_in, const std::vector<HUniv>& u_in, int root,
                const BuildOpts& opts, Flat& F);

}  // namespace nt
