// Device geometry layout shared by the host builder (builder.cpp) and the kernels
// (track.cu).  Everything is flattened into one contiguous device blob of plain
// arrays (SoA where the access pattern is per-field, small AoS records where a
// whole record is consumed at once).  DESIGN.md "Data layout" documents it.
#pragma once
#include <cstddef>
#include <cstdint>

#ifdef __CUDACC__
#define NT_HD __host__ __device__ __forceinline__
#else
#define NT_HD inline
#endif

// Device code is compiled once per feature set (track_f0.cu: rect/CSG models with axis planes and
// cylinders only; track_f7.cu: everything) into namespace nt::NT_NS, so a model that uses no hex
// arrays, general planes or spheres runs a kernel without that code (smaller i-cache footprint).
#ifndef NT_NS
#define NT_NS fall
#endif
#ifndef NT_FEAT
#define NT_FEAT 7
#endif
#define NT_DEV_BEGIN namespace nt { namespace NT_NS {
#define NT_DEV_END } }

namespace nt {

enum Feature : int { F_HEX = 1, F_PLANE = 2, F_SPHERE = 4, F_RECTNU = 8 };   // F_RECTNU: non-uniform rect

constexpr int kMaxDepth = 8;          // builder-enforced nesting limit (reading O7)
constexpr int kBihStack = 12;         // BIH depth limit = register stack capacity (nt_geom.cuh)
constexpr int kNC = 18;               // counters (NT_NC)
constexpr double kFlagDist = 1e-10;   // O16 proximity / near-tie distance (cm)
constexpr double kHexH = 0.8660254037844386;  // O9: nearest double to sqrt(3)/2

enum SurfKind : int { S_PX = 0, S_PY = 1, S_PZ = 2, S_PLANE = 3, S_CZ = 4, S_SPHERE = 5 };
enum UnivKind : int { U_CSG = 0, U_RECT = 1, U_HEX = 2 };

// Surface record: 32 bytes.  PX/PY/PZ: c0 = a.  PLANE: nx, ny, nz, d.
// CZ: x0, y0, R*R (c3 unused).  SPHERE: x0, y0, z0, R*R.
struct alignas(16) DSurf { double c[4]; };

// Half-space record (48 bytes): the cell's packed entry with its surface's coefficients, O16
// tolerance and surf_meta (kind | bc << 4) copied in, so that a distance, containment or crossing
// step loads everything from one index (no dependent hs -> surface load).  hsr[h] mirrors hs[h].
// A CSG distance winner is identified by its half-space index h (Best::j), which also names the
// crossed surface's neighbour list (hs_nb_off[h]) for the descent.
struct alignas(16) DHs { double c[4]; int32_t e, meta; double tol; };
// DHs::meta bit above surf_meta: this entry and the next form a slab (same axis plane kind, opposite
// senses), evaluated together by the distance loop
constexpr int32_t kHsSlab = 0x100;

// Half-space entry of a cell: (sid << 4) | (kind << 1) | sense  (sense 1 = positive side).
NT_HD int hs_sid(int h) { return h >> 4; }
NT_HD int hs_kind(int h) { return (h >> 1) & 7; }
NT_HD int hs_sense(int h) { return h & 1; }
inline int hs_pack(int sid, int kind, int sense) { return (sid << 4) | (kind << 1) | sense; }

// Universe record (160 bytes).
//  CSG : i0 = BIH root node, i1 = first cell, i2 = cell count
//  RECT: i0..i2 = shape, is2d; d[0..2] = lower-left, d[3..5] = pitch
//  HEX : i0 = R = rings-1, i1 = nz (0 = 2-D), i2 = orient; ntile = (2R+1)^2
//        d[0..1] = C, d[2] = pitch, d[3] = pitch*H, d[4] = z_lower, d[5] = z_pitch,
//        d[6..7] = a1, d[8..9] = a2, d[10..15] = n0x n0y n1x n1y n2x n2y
//  fill_off: offset into `fills` (RECT: shape product entries, x fastest;
//            HEX: ntile * max(nz,1) entries indexed (r+R)*(2R+1)+(q+R) + kz*ntile;
//            -1 entries = out of lattice -> outer), outer: universe id or -1.
struct alignas(16) DUniv {
  int32_t kind, i0, i1, i2;
  int32_t fill_off, outer, is2d, ntile;   // rect: ntile = offset of the edge table (N1), -1 uniform
  double d[16];
};

// Cell reference (16 bytes) as listed by BIH leaves and crossing-neighbour lists: the cell id with its
// fill (material-cell bin >= 0, or -1 - daughter uid) and its half-space range [h0, h1), so that a
// point-location step reads everything about a candidate cell with one 16-byte load.
struct alignas(16) CRef { int32_t cell, fill, h0, h1; };

// Bounding-interval-hierarchy node (24 bytes): two planes per node.
//  meta >= 0: internal, split axis = meta, children a and a+1;
//             left child covers x[axis] <= lmax, right child x[axis] >= rmin (may overlap).
//  meta <  0: leaf with (-meta - 1) cells at bih_leaf[a ..].
struct BihNode { double lmax, rmin; int32_t meta, a; };

// Everything a kernel needs, passed by value (kernel parameter space).
struct DevGeom {
  const DSurf* surf;
  const double* surf_tol;     // O16 proximity tolerance per surface
  const uint8_t* surf_meta;   // per surface: kind | (nt_bc << 4)
  const int32_t* hs;          // packed half-spaces, per cell sorted by surface id (O13)
  const DHs* hsr;             // per half-space entry: packed entry + surface coefficients + tolerance
  const int32_t* cell_hs;     // [n_cells+1] CSR offsets into hs
  const int32_t* cell_fill;   // >= 0: material-cell index (tally bin); < 0: -1 - daughter uid
  const double* cell_tr;      // [3*n_cells] fill translation
  const DUniv* univ;
  const BihNode* bih;
  const CRef* bih_leaf;       // leaf cell lists (cell references)
  const int32_t* fills;
  const double* mc_st;        // per material cell: sigma_t
  const double* mc_pabs;      // per material cell: sigma_a / sigma_t (O14)
  const double* mc_nut;       // per material cell: nu Sigma_f / Sigma_a (F1)
  const int32_t* mc_cell;     // per material cell: global cell id (trace)
  const double* edges;        // non-uniform rect edges (N1): per array x[n0+1] y[n1+1] z[n2+1]
  const int32_t* univ_inst;   // per-instance tallies (D1): per universe, base into inst_off
  const int32_t* inst_off;    //   instances before child k of the universe
  const int32_t* cell_pos;    //   per cell: its position in its universe
  const int32_t* hs_nb_off;   // per half-space entry: [off, off+1) into nb_cells (CSG crossing shortcut)
  const CRef* nb_cells;       // cell references
  int32_t root, n_mc, max_depth, n_univ;
  int32_t n_cells, n_surf, root_kind, features;   // features: F_* bits present in the model
  const void* const* trk;     // DP dispatch only: per-universe tracker object pointers (dp_tracker.cuh)
  void* pool;                 // host use only: the model's own cudaMemPool_t for per-launch scratch
  double mesh_lo[3], mesh_d[3];   // superimposed mesh (M1): voxel edges lo + i d
  int32_t mesh_n[3], mesh_on;
  int32_t max_sites;              // F1: sites one absorption can bank
};

// Rect-specialised tracker tables (Alg. 9-10): root = axis box or concentric CZ annuli between a
// PZ pair, then K rect levels, then a concentric-CZ pin.  Surfaces are read from the generic
// DSurf table (same arithmetic); rect universes from the DUniv table.
struct RectGeom {
  int32_t K;                 // number of rect levels (0..4)
  int32_t root_box;          // 1: root cell is an axis box; 0: CZ annuli + PZ pair
  int32_t root_fill_cell;    // root cell holding level 1 (box cell / innermost annulus)
  int32_t n_root_cells;      // CZ root: number of annuli
  int32_t root_univ_child;   // universe id of level 1
  int32_t box_sid[6];        // box root: PX-, PX+, PY-, PY+, PZ-, PZ+ surface ids
  int32_t zsid[2];           // CZ root: lower / upper PZ surface ids
  int32_t root_sid[16];      // annulus k: outer CZ surface id (inner one = root_sid[k-1])
  int32_t root_cell[16];     // annulus k: global cell id
  int32_t root_mc[16];       // annulus k: material-cell index (-1 for the core annulus)
  const int32_t* pin_of_univ;  // per universe: pin index or -1
  const int32_t* pin_off;      // [n_pins+1] offsets into pin_sid (pin p has off[p+1]-off[p] CZs)
  const int32_t* pin_sid;      // pin CZ surface ids, ascending radius
  const int32_t* pin_mc;       // material-cell index of annulus k of pin p at pin_off[p] + p + k
};

}  // namespace nt
