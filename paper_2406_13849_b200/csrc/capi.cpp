// extern "C" boundary of libnestrack.so (include/nestrack.h): argument checking, status
// codes, thread-local error text, the device copy of the model, and kernel launches.
#include <cuda_runtime.h>

#include <atomic>
#include <cmath>
#include <cstring>
#include <mutex>
#include <new>
#include <string>
#include <vector>

#include "../../include/nestrack.h"
#include "nt_model.hpp"

#include "nt_kernels.hpp"

using namespace nt;

static thread_local std::string g_err;

static nt_status err(nt_status s, const std::string& msg) {
  g_err = msg;
  return s;
}
static nt_status cuda_err(cudaError_t e, const char* where) {
  return err(NT_E_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

constexpr int kSlots = 64;

struct nt_model {
  std::vector<HSurf> s;
  std::vector<HMat> m;
  std::vector<HCell> c;
  std::vector<HUniv> u;
  int root = -1;
  bool finalized = false;
  BuildOpts opts;
  Flat F;
  // device
  int device = -1;
  void* blob = nullptr;
  size_t blob_bytes = 0;
  DevGeom g{};
  RectGeom rg{};
  unsigned long long* counters = nullptr;   // kSlots work counters
  std::atomic<unsigned> slot{0};
  double* host_scratch_dev = nullptr;       // nt_track_host device output
  size_t host_scratch_len = 0;
  std::mutex host_mu;
  int last_launches = 0;
  void* dp_objs = nullptr;                  // DP dispatch: tracker objects + pointer table (lazy)
  cudaMemPool_t pool = nullptr;             // per-launch scratch (stream-ordered), owned by the model
  bool mesh_on = false;                     // superimposed mesh (M1)
  double mesh_lo[3] = {0, 0, 0}, mesh_d[3] = {0, 0, 0};
  int32_t mesh_n[3] = {0, 0, 0};
  std::mutex dp_mu;
};

// Coefficients of the spec'd transcendentals (reading R-T), computed with IEEE double ops.
static void coef_table(double* c) {
  for (int k = 0; k <= 11; ++k) c[k] = 1.0 / (double)(2 * k + 1);
  double fact[20];
  fact[0] = 1.0;
  for (int k = 1; k < 20; ++k) fact[k] = fact[k - 1] * (double)k;
  for (int k = 1; k <= 9; ++k) {
    const double sk = 1.0 / fact[2 * k + 1], ck = 1.0 / fact[2 * k];
    c[12 + k - 1] = (k & 1) ? -sk : sk;
    c[21 + k - 1] = (k & 1) ? -ck : ck;
  }
}

template <class T>
static size_t place(std::vector<char>& blob, const std::vector<T>& v) {
  size_t off = (blob.size() + 255) & ~size_t(255);
  blob.resize(off + v.size() * sizeof(T));
  if (!v.empty()) std::memcpy(blob.data() + off, v.data(), v.size() * sizeof(T));
  return off;
}

extern "C" {

const char* nt_last_error(void) { return g_err.c_str(); }
int32_t nt_abi_version(void) { return NT_ABI_VERSION; }

nt_status nt_model_create(nt_model** out) {
  if (!out) return err(NT_E_ARG, "nt_model_create: out is NULL");
  *out = new (std::nothrow) nt_model();
  if (!*out) return err(NT_E_NOMEM, "nt_model_create: out of host memory");
  return NT_OK;
}

// frees every device resource of the model (on its device; the caller selects it)
static void release_device(nt_model* m) {
  if (m->blob) cudaFree(m->blob);
  if (m->counters) cudaFree(m->counters);
  if (m->host_scratch_dev) cudaFree(m->host_scratch_dev);
  if (m->dp_objs) cudaFree(m->dp_objs);
  if (m->pool) cudaMemPoolDestroy(m->pool);    // outstanding stream-ordered frees complete first
  m->blob = nullptr; m->counters = nullptr; m->host_scratch_dev = nullptr; m->dp_objs = nullptr;
  m->pool = nullptr;
}

void nt_model_destroy(nt_model* m) {
  if (!m) return;
  if (m->blob || m->counters || m->host_scratch_dev || m->dp_objs || m->pool) {
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(m->device);
    release_device(m);
    cudaSetDevice(prev);
  }
  delete m;
}

#define CHECK_BUILDER(m)                                                        \
  do {                                                                          \
    if (!(m)) return err(NT_E_ARG, std::string(__func__) + ": model is NULL");  \
    if ((m)->finalized) return err(NT_E_ORDER, std::string(__func__) + ": model already finalized"); \
  } while (0)

nt_status nt_add_surface(nt_model* m, nt_surface_kind kind, const double* coef, nt_bc bc, int32_t* id) {
  CHECK_BUILDER(m);
  if (!coef) return err(NT_E_ARG, "nt_add_surface: coef is NULL");
  if ((int)kind < 0 || (int)kind > NT_SPHERE) return err(NT_E_ARG, "nt_add_surface: bad kind");
  if ((int)bc < 0 || (int)bc > NT_BC_REFLECT) return err(NT_E_ARG, "nt_add_surface: bad bc");
  HSurf s{(int)kind, (int)bc, {0, 0, 0, 0}};
  const int nco = kind <= NT_PZ ? 1 : (kind == NT_CZ ? 3 : 4);
  for (int i = 0; i < nco; ++i) s.c[i] = coef[i];
  m->s.push_back(s);
  if (id) *id = (int32_t)m->s.size() - 1;
  return NT_OK;
}

nt_status nt_add_material(nt_model* m, double st, double sa, int32_t* id) {
  CHECK_BUILDER(m);
  m->m.push_back({st, sa, 0.0});
  if (id) *id = (int32_t)m->m.size() - 1;
  return NT_OK;
}

nt_status nt_set_fission(nt_model* m, int32_t mat, double nu_sigma_f) {
  CHECK_BUILDER(m);
  if (mat < 0 || mat >= (int)m->m.size()) return err(NT_E_ID, "nt_set_fission: material id out of range");
  m->m[mat].nusf = nu_sigma_f;        // validated at nt_finalize
  return NT_OK;
}

nt_status nt_add_csg_universe(nt_model* m, int32_t* uid) {
  CHECK_BUILDER(m);
  HUniv u;
  u.kind = U_CSG;
  m->u.push_back(u);
  if (uid) *uid = (int32_t)m->u.size() - 1;
  return NT_OK;
}

nt_status nt_add_cell(nt_model* m, int32_t uid, const int32_t* hs, int32_t n, nt_fill_kind fk,
                      int32_t fill, const double tr[3], int32_t* cell_id) {
  CHECK_BUILDER(m);
  if (uid < 0 || uid >= (int)m->u.size()) return err(NT_E_ID, "nt_add_cell: universe id out of range");
  if (m->u[uid].kind != U_CSG) return err(NT_E_ARG, "nt_add_cell: universe is not a CSG universe");
  if (n < 0 || (n > 0 && !hs)) return err(NT_E_ARG, "nt_add_cell: bad half-space list");
  if ((int)fk != 0 && (int)fk != 1) return err(NT_E_ARG, "nt_add_cell: bad fill kind");
  HCell c;
  c.uid = uid;
  for (int i = 0; i < n; ++i) {
    if (hs[i] == 0) return err(NT_E_ARG, "nt_add_cell: half-space 0 is invalid (use +-(surf+1))");
    c.sid.push_back((hs[i] > 0 ? hs[i] : -hs[i]) - 1);
    c.sense.push_back(hs[i] > 0 ? 1 : 0);
  }
  c.fill_kind = (int)fk;
  c.fill = fill;
  for (int a = 0; a < 3; ++a) c.tr[a] = tr ? tr[a] : 0.0;
  m->c.push_back(c);
  m->u[uid].cells.push_back((int)m->c.size() - 1);
  if (cell_id) *cell_id = (int32_t)m->c.size() - 1;
  return NT_OK;
}

nt_status nt_add_rect_array(nt_model* m, const double ll[3], const double p[3], const int32_t shape[3],
                            const int32_t* fill, int32_t outer, int32_t* uid) {
  CHECK_BUILDER(m);
  if (!ll || !p || !shape || !fill) return err(NT_E_ARG, "nt_add_rect_array: NULL argument");
  HUniv u;
  u.kind = U_RECT;
  for (int a = 0; a < 3; ++a) { u.ll[a] = ll[a]; u.p[a] = p[a]; u.n[a] = shape[a]; }
  u.is2d = p[2] == 0.0;
  if (u.is2d) u.n[2] = 1;
  for (int a = 0; a < 3; ++a)
    if (u.n[a] < 1 || u.n[a] > (1 << 20)) return err(NT_E_GEOMETRY, "nt_add_rect_array: bad shape");
  const long n = (long)u.n[0] * u.n[1] * u.n[2];
  u.fill.assign(fill, fill + n);
  u.outer = outer;
  m->u.push_back(u);
  if (uid) *uid = (int32_t)m->u.size() - 1;
  return NT_OK;
}

nt_status nt_add_rect_edges(nt_model* m, const double* edges, const int32_t n_edges[3], const int32_t* fill,
                            int32_t outer, int32_t* uid) {
  CHECK_BUILDER(m);
  if (!edges || !n_edges || !fill) return err(NT_E_ARG, "nt_add_rect_edges: NULL argument");
  HUniv u;
  u.kind = U_RECT;
  u.is2d = n_edges[2] == 0;
  long off = 0;
  for (int a = 0; a < 3; ++a) {
    if (n_edges[a] < 0 || n_edges[a] > (1 << 20) || (a < 2 && n_edges[a] < 2) || (a == 2 && n_edges[a] == 1))
      return err(NT_E_GEOMETRY, "nt_add_rect_edges: need >= 2 edges per axis (z: 0 for 2-D)");
    u.e[a].assign(edges + off, edges + off + n_edges[a]);
    off += n_edges[a];
    u.n[a] = n_edges[a] > 0 ? n_edges[a] - 1 : 1;
    u.ll[a] = n_edges[a] > 0 ? edges[off - n_edges[a]] : 0.0;
  }
  const long n = (long)u.n[0] * u.n[1] * u.n[2];
  u.fill.assign(fill, fill + n);
  u.outer = outer;
  m->u.push_back(u);
  if (uid) *uid = (int32_t)m->u.size() - 1;
  return NT_OK;
}

nt_status nt_add_hex_array(nt_model* m, nt_hex_orient orient, const double center[2], double pitch,
                           int32_t rings, double zlo, double zp, int32_t nz, const int32_t* fill,
                           int32_t outer, int32_t* uid) {
  CHECK_BUILDER(m);
  if (!center || !fill) return err(NT_E_ARG, "nt_add_hex_array: NULL argument");
  if ((int)orient != 0 && (int)orient != 1) return err(NT_E_ARG, "nt_add_hex_array: bad orientation");
  if (rings < 1 || rings > 1000) return err(NT_E_GEOMETRY, "nt_add_hex_array: bad ring count");
  HUniv u;
  u.kind = U_HEX;
  u.orient = (int)orient;
  u.C[0] = center[0];
  u.C[1] = center[1];
  u.pitch = pitch;
  u.rings = rings;
  u.zlo = zlo;
  u.zp = zp;
  u.nz = zp > 0 ? nz : 0;
  if (zp > 0 && nz < 1) return err(NT_E_GEOMETRY, "nt_add_hex_array: nz must be >= 1 with z_pitch > 0");
  const long ntile = 1 + 3L * rings * (rings - 1);
  u.fill.assign(fill, fill + ntile * (u.nz > 0 ? u.nz : 1));
  u.outer = outer;
  m->u.push_back(u);
  if (uid) *uid = (int32_t)m->u.size() - 1;
  return NT_OK;
}

nt_status nt_set_root(nt_model* m, int32_t uid) {
  CHECK_BUILDER(m);
  if (uid < 0 || uid >= (int)m->u.size()) return err(NT_E_ID, "nt_set_root: universe id out of range");
  m->root = uid;
  return NT_OK;
}

nt_status nt_set_mesh(nt_model* m, const double lo[3], const double hi[3], const int32_t shape[3]) {
  CHECK_BUILDER(m);
  if (!lo || !hi || !shape) return err(NT_E_ARG, "nt_set_mesh: NULL argument");
  for (int a = 0; a < 3; ++a)
    if (shape[a] < 1 || shape[a] > 4096 || !(hi[a] > lo[a]) || !std::isfinite(lo[a]) || !std::isfinite(hi[a]))
      return err(NT_E_GEOMETRY, "nt_set_mesh: need 1 <= shape <= 4096 and finite lo < hi on every axis");
  for (int a = 0; a < 3; ++a) {
    m->mesh_lo[a] = lo[a];
    m->mesh_d[a] = (hi[a] - lo[a]) / (double)shape[a];
    m->mesh_n[a] = shape[a];
  }
  m->mesh_on = true;
  return NT_OK;
}

void nt_build_opts_default(nt_build_opts* o) {
  if (!o) return;
  o->device = 0;
  o->bih_max_leaf = 4;
  o->pseudo_array = 0;
  o->reserved = 0;
  o->sah_ct = 1.0;
  o->sah_ci = 1.0;
}

nt_status nt_finalize(nt_model* m, const nt_build_opts* o) {
  CHECK_BUILDER(m);
  nt_build_opts d;
  nt_build_opts_default(&d);
  if (!o) o = &d;
  m->opts.device = o->device;
  m->opts.max_leaf = o->bih_max_leaf > 0 ? o->bih_max_leaf : 4;
  m->opts.pseudo = o->pseudo_array;
  m->opts.ct = o->sah_ct > 0 ? o->sah_ct : 1.0;
  m->opts.ci = o->sah_ci > 0 ? o->sah_ci : 1.0;
  try {
    build_flat(m->s, m->m, m->c, m->u, m->root, m->opts, m->F);
  } catch (const GeomError& e) {
    return err(NT_E_GEOMETRY, std::string("nt_finalize: ") + e.what());
  } catch (const std::bad_alloc&) {
    return err(NT_E_NOMEM, "nt_finalize: out of host memory");
  }
  const Flat& F = m->F;
  // leaf and neighbour lists as cell references (cell, fill, half-space range)
  auto cref = [&F](const std::vector<int32_t>& ids) {
    std::vector<CRef> r(ids.size());
    for (size_t i = 0; i < ids.size(); ++i) {
      const int c = ids[i];
      const bool ok = c >= 0 && c < (int)F.cell_fill.size();
      r[i] = ok ? CRef{c, F.cell_fill[c], F.cell_hs[c], F.cell_hs[c + 1]} : CRef{c, 0, 0, 0};
    }
    return r;
  };
  const std::vector<CRef> leaf_refs = cref(F.bih_leaf), nb_refs = cref(F.nb_cells);
  // one contiguous blob of 256-byte aligned arrays
  std::vector<char> blob;
  const size_t o_surf = place(blob, F.surf), o_tol = place(blob, F.surf_tol), o_meta = place(blob, F.surf_meta),
               o_hs = place(blob, F.hs), o_chs = place(blob, F.cell_hs), o_cf = place(blob, F.cell_fill),
               o_ctr = place(blob, F.cell_tr), o_univ = place(blob, F.univ), o_bih = place(blob, F.bih),
               o_leaf = place(blob, leaf_refs), o_fills = place(blob, F.fills), o_st = place(blob, F.mc_st),
               o_pabs = place(blob, F.mc_pabs), o_mcc = place(blob, F.mc_cell), o_nut = place(blob, F.mc_nut),
               o_edges = place(blob, F.edges), o_uinst = place(blob, F.univ_inst),
               o_ioff = place(blob, F.inst_off), o_cpos = place(blob, F.cell_pos),
               o_nboff = place(blob, F.hs_nb_off), o_nbc = place(blob, nb_refs), o_hsr = place(blob, F.hsr);
  const size_t o_pou = place(blob, F.r_pin_of_univ), o_poff = place(blob, F.r_pin_off),
               o_psid = place(blob, F.r_pin_sid), o_pmc = place(blob, F.r_pin_mc);
  m->blob_bytes = blob.size();
  m->device = o->device;
  if (o->device >= 0) {
    int prev = 0;
    cudaGetDevice(&prev);
    cudaError_t e = cudaSetDevice(o->device);
    if (e != cudaSuccess) return cuda_err(e, "nt_finalize: cudaSetDevice");
    {   // per-launch scratch is stream-ordered, from a memory pool the model owns (not the device's
        // default pool, which other users of cudaMallocAsync share): it keeps up to 64 MB across
        // synchronisations instead of unmapping and remapping the scratch every launch
      cudaMemPoolProps props{};
      props.allocType = cudaMemAllocationTypePinned;
      props.location.type = cudaMemLocationTypeDevice;
      props.location.id = o->device;
      cudaMemPool_t pool = nullptr;
      e = cudaMemPoolCreate(&pool, &props);
      if (e != cudaSuccess) { cudaSetDevice(prev); return cuda_err(e, "nt_finalize: cudaMemPoolCreate"); }
      uint64_t keep = 64ull << 20;
      e = cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
      if (e != cudaSuccess) { cudaMemPoolDestroy(pool); cudaSetDevice(prev); return cuda_err(e, "nt_finalize: pool"); }
      m->pool = pool;
    }
    e = cudaMalloc(&m->blob, blob.size());
    if (e != cudaSuccess) { release_device(m); cudaSetDevice(prev); return cuda_err(e, "nt_finalize: cudaMalloc"); }
    e = cudaMemcpy(m->blob, blob.data(), blob.size(), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMalloc(&m->counters, sizeof(unsigned long long) * kSlots);
    if (e == cudaSuccess) e = cudaMemset(m->counters, 0, sizeof(unsigned long long) * kSlots);
    double coef[30];
    coef_table(coef);
    if (e == cudaSuccess) e = f0::upload_coefficients(coef, 30);
    if (e == cudaSuccess) e = f7::upload_coefficients(coef, 30);
    if (e == cudaSuccess) e = f0r::upload_coefficients(coef, 30);
    if (e == cudaSuccess) e = fh::upload_coefficients(coef, 30);
    if (e != cudaSuccess) release_device(m);     // a failed finalize leaves nothing behind
    cudaSetDevice(prev);
    if (e != cudaSuccess) return cuda_err(e, "nt_finalize: upload");
    char* b = static_cast<char*>(m->blob);
    DevGeom& g = m->g;
    g.pool = m->pool;
    g.surf = (const DSurf*)(b + o_surf);
    g.surf_tol = (const double*)(b + o_tol);
    g.surf_meta = (const uint8_t*)(b + o_meta);
    g.hs = (const int32_t*)(b + o_hs);
    g.hsr = (const DHs*)(b + o_hsr);
    g.cell_hs = (const int32_t*)(b + o_chs);
    g.cell_fill = (const int32_t*)(b + o_cf);
    g.cell_tr = (const double*)(b + o_ctr);
    g.univ = (const DUniv*)(b + o_univ);
    g.bih = (const BihNode*)(b + o_bih);
    g.bih_leaf = (const CRef*)(b + o_leaf);
    g.fills = (const int32_t*)(b + o_fills);
    g.mc_st = (const double*)(b + o_st);
    g.mc_pabs = (const double*)(b + o_pabs);
    g.mc_nut = (const double*)(b + o_nut);
    g.mc_cell = (const int32_t*)(b + o_mcc);
    g.edges = (const double*)(b + o_edges);
    g.univ_inst = (const int32_t*)(b + o_uinst);
    g.inst_off = (const int32_t*)(b + o_ioff);
    g.cell_pos = (const int32_t*)(b + o_cpos);
    g.hs_nb_off = (const int32_t*)(b + o_nboff);
    g.nb_cells = (const CRef*)(b + o_nbc);
    m->rg = F.rg;
    m->rg.pin_of_univ = (const int32_t*)(b + o_pou);
    m->rg.pin_off = (const int32_t*)(b + o_poff);
    m->rg.pin_sid = (const int32_t*)(b + o_psid);
    m->rg.pin_mc = (const int32_t*)(b + o_pmc);
  }
  DevGeom& g = m->g;
  g.root = F.root;
  g.n_mc = F.n_mc;
  g.max_depth = F.max_depth;
  g.n_univ = (int)F.univ.size();
  g.n_cells = (int)F.cell_fill.size();
  g.n_surf = (int)F.surf.size();
  g.root_kind = F.univ[F.root].kind;
  g.features = F.features;
  g.mesh_on = m->mesh_on ? 1 : 0;
  g.max_sites = F.max_sites;
  for (int a = 0; a < 3; ++a) { g.mesh_lo[a] = m->mesh_lo[a]; g.mesh_d[a] = m->mesh_d[a]; g.mesh_n[a] = m->mesh_n[a]; }
  m->finalized = true;
  return NT_OK;
}

nt_status nt_model_info_get(const nt_model* m, nt_model_info* info) {
  if (!m || !info) return err(NT_E_ARG, "nt_model_info_get: NULL argument");
  if (!m->finalized) return err(NT_E_ORDER, "nt_model_info_get: model not finalized");
  const Flat& F = m->F;
  info->n_surfaces = (int)F.surf.size();
  info->n_cells = (int)F.cell_fill.size();
  info->n_material_cells = F.n_mc;
  info->n_universes = (int)F.univ.size();
  info->max_depth = F.max_depth;
  info->rect_specialisable = F.rect_ok ? 1 : 0;
  info->rect_levels = F.rect_K;
  info->n_bih_nodes = (int)F.bih.size();
  info->out_len = 2 * (int64_t)F.n_mc + NT_NC;
  info->device_bytes = m->blob_bytes;
  info->mesh_bins = m->mesh_on ? (int64_t)m->mesh_n[0] * m->mesh_n[1] * m->mesh_n[2] : 0;
  info->n_instances = F.n_inst;
  info->max_sites = F.max_sites;
  return NT_OK;
}

nt_status nt_fission_source(nt_model* m, const double* d_bank, const uint8_t* d_bank_n, uint64_t n_prev,
                            uint64_t seed, uint32_t cycle, uint64_t n_next, double* d_states,
                            uint64_t* total_sites, void* stream) {
  if (!m || !total_sites || (n_prev && (!d_bank || !d_bank_n)) || (n_next && !d_states))
    return err(NT_E_ARG, "nt_fission_source: NULL argument");
  if (!m->finalized || !m->blob) return err(NT_E_ORDER, "nt_fission_source: model not finalized on a device");
  int prev = 0;
  cudaGetDevice(&prev);
  if (prev != m->device) cudaSetDevice(m->device);
  unsigned long long M = 0;
  const bool f0 = m->g.features == 0;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaError_t e = f0 ? f0::fission_source(m->g, d_bank, d_bank_n, n_prev, seed, cycle, n_next, d_states, &M, s)
                     : f7::fission_source(m->g, d_bank, d_bank_n, n_prev, seed, cycle, n_next, d_states, &M, s);
  if (prev != m->device) cudaSetDevice(prev);
  if (e != cudaSuccess) return cuda_err(e, "nt_fission_source");
  *total_sites = M;
  m->last_launches = M ? 5 : 3;
  return NT_OK;
}

nt_status nt_bank_compact(nt_model* m, const double* d_bank, const uint8_t* d_bank_n, uint64_t n, double* d_sites,
                          uint64_t* total_sites, void* stream) {
  if (!m || !total_sites || (n && (!d_bank || !d_bank_n || !d_sites)))
    return err(NT_E_ARG, "nt_bank_compact: NULL argument");
  if (!m->finalized || !m->blob) return err(NT_E_ORDER, "nt_bank_compact: model not finalized on a device");
  int prev = 0;
  cudaGetDevice(&prev);
  if (prev != m->device) cudaSetDevice(m->device);
  unsigned long long M = 0;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaError_t e = m->g.features == 0 ? f0::bank_compact(m->g, d_bank, d_bank_n, n, d_sites, &M, s)
                                     : f7::bank_compact(m->g, d_bank, d_bank_n, n, d_sites, &M, s);
  if (prev != m->device) cudaSetDevice(prev);
  if (e != cudaSuccess) return cuda_err(e, "nt_bank_compact");
  *total_sites = M;
  return NT_OK;
}

nt_status nt_source_from_sites(nt_model* m, const double* d_sites, uint64_t total_sites, uint64_t seed,
                               uint32_t cycle, uint64_t j_begin, uint64_t n_next, double* d_states, void* stream) {
  if (!m || (total_sites && !d_sites) || (n_next && !d_states)) return err(NT_E_ARG, "nt_source_from_sites: NULL argument");
  if (!m->finalized || !m->blob) return err(NT_E_ORDER, "nt_source_from_sites: model not finalized on a device");
  if (total_sites == 0 && n_next) return err(NT_E_ARG, "nt_source_from_sites: no sites (subcritical collapse)");
  int prev = 0;
  cudaGetDevice(&prev);
  if (prev != m->device) cudaSetDevice(m->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaError_t e = m->g.features == 0 ? f0::source_from_sites(d_sites, total_sites, seed, cycle, j_begin, n_next, d_states, s)
                                     : f7::source_from_sites(d_sites, total_sites, seed, cycle, j_begin, n_next, d_states, s);
  if (prev != m->device) cudaSetDevice(prev);
  if (e != cudaSuccess) return cuda_err(e, "nt_source_from_sites");
  m->last_launches = 1;
  return NT_OK;
}

nt_status nt_instance_cells(const nt_model* m, int32_t* out, int64_t cap) {
  if (!m || !out) return err(NT_E_ARG, "nt_instance_cells: NULL argument");
  if (!m->finalized) return err(NT_E_ORDER, "nt_instance_cells: model not finalized");
  for (int64_t i = 0; i < m->F.n_inst && i < cap; ++i) out[i] = m->F.inst_mc[(size_t)i];
  return NT_OK;
}

nt_status nt_material_cell_ids(const nt_model* m, int32_t* out, int32_t cap) {
  if (!m || (!out && cap > 0)) return err(NT_E_ARG, "nt_material_cell_ids: NULL argument");
  if (!m->finalized) return err(NT_E_ORDER, "nt_material_cell_ids: model not finalized");
  for (int i = 0; i < m->F.n_mc && i < cap; ++i) out[i] = m->F.mc_cell[i];
  return NT_OK;
}

nt_status nt_bih_info(const nt_model* m, int32_t uid, int32_t* n_nodes, int32_t* depth, int32_t* leaf_cells,
                      int32_t cap, int32_t* n_leaf_cells) {
  if (!m) return err(NT_E_ARG, "nt_bih_info: model is NULL");
  if (!m->finalized) return err(NT_E_ORDER, "nt_bih_info: model not finalized");
  if (uid < 0 || uid >= (int)m->F.univ.size()) return err(NT_E_ID, "nt_bih_info: universe id out of range");
  const DUniv& U = m->F.univ[uid];
  if (U.kind != U_CSG) return err(NT_E_ARG, "nt_bih_info: not a CSG universe");
  // walk the subtree
  std::vector<int> todo{U.i0};
  int nodes = 0, cnt = 0;
  while (!todo.empty()) {
    const int n = todo.back();
    todo.pop_back();
    ++nodes;
    const BihNode& b = m->F.bih[n];
    if (b.meta < 0) {
      for (int q = 0; q < -b.meta - 1; ++q) {
        if (leaf_cells && cnt < cap) leaf_cells[cnt] = m->F.bih_leaf[b.a + q];
        ++cnt;
      }
    } else {
      todo.push_back(b.a + 1);
      todo.push_back(b.a);
    }
  }
  if (n_nodes) *n_nodes = nodes;
  if (depth) *depth = m->F.bih_depth[uid];
  if (n_leaf_cells) *n_leaf_cells = cnt;
  return NT_OK;
}

static nt_status run_common(nt_model* m, const nt_run* run, const double* d_states, const nt_outputs* o,
                            void* stream, const char* who) {
  if (!m || !run || !o) return err(NT_E_ARG, std::string(who) + ": NULL argument");
  if (!m->finalized) return err(NT_E_ORDER, std::string(who) + ": model not finalized");
  if (m->device < 0 || !m->blob) return err(NT_E_ORDER, std::string(who) + ": host-only model (device = -1)");
  if (!o->out) return err(NT_E_ARG, std::string(who) + ": outputs.out is NULL");
  const bool trace = (run->flags & NT_TRACE) != 0;
  if (trace && (!o->trace_count || (!o->trace && o->trace_cap))) return err(NT_E_ARG, std::string(who) + ": trace buffers");
  if (run->tracker != NT_TRACKER_GENERIC && run->tracker != NT_TRACKER_RECT)
    return err(NT_E_ARG, std::string(who) + ": bad tracker");
  if (run->tracker == NT_TRACKER_RECT && !m->F.rect_ok)
    return err(NT_E_UNSUPPORTED, std::string(who) + ": model is not rect-specialisable: " + m->F.rect_why);
  if (run->tracker == NT_TRACKER_RECT && (run->flags & (NT_WARPQ | NT_ROUNDS | NT_DP)))
    return err(NT_E_ARG, std::string(who) + ": the rect tracker runs on the ring queues (default) or history-based "
               "(NT_HISTORY)");
  if (run->max_segments > 0xFFFFFFFFull) return err(NT_E_ARG, std::string(who) + ": max_segments >= 2^32");
  const int block = run->block_dim > 0 ? run->block_dim : 256;
  if (block % 32 || block > 256) return err(NT_E_ARG, std::string(who) + ": block_dim must be a multiple of 32, <= 256");
  if (run->tracker == NT_TRACKER_GENERIC && !(run->flags & (NT_WARPQ | NT_HISTORY)) && block != 128 && block != 256 &&
      !(block == 192 && !(run->flags & (NT_ROUNDS | NT_DP))))
    return err(NT_E_ARG, std::string(who) + ": the event scheduler needs block_dim 128 or 256 (192: ring queues, SP only)");
  if (run->n > 0xFFFFFFFFull) return err(NT_E_ARG, std::string(who) + ": at most 2^32-1 histories per call");
  if (trace && o->mesh && m->mesh_on)
    return err(NT_E_UNSUPPORTED, std::string(who) + ": the mesh tally cannot be combined with NT_TRACE");
  if (o->inst && (trace || m->F.n_inst == 0 || run->tracker == NT_TRACKER_RECT))
    return err(NT_E_UNSUPPORTED, std::string(who) + ": instance tallies need a generic-tracker run without "
               "NT_TRACE on a model built without pseudo-arrays");
  const bool dp = (run->flags & NT_DP) != 0;
  // block queues: ring queues without rounds (default, block 256) or rounds + barrier (NT_ROUNDS,
  // also every block_dim 128 run)
  const bool async = !(run->flags & NT_ROUNDS) && (block == 256 || block == 192);
  if (dp && (run->tracker != NT_TRACKER_GENERIC || (run->flags & (NT_WARPQ | NT_HISTORY)) || block != 256))
    return err(NT_E_ARG, std::string(who) + ": NT_DP needs the generic tracker, block queues and block_dim 256");
  m->last_launches = 0;
  if (run->n == 0) return NT_OK;
  int prev = 0;
  cudaGetDevice(&prev);
  if (prev != m->device) cudaSetDevice(m->device);
  KRun R{};
  R.seed = run->seed;
  R.pid0 = run->pid_begin;
  R.n = run->n;
  R.max_seg = run->max_segments ? run->max_segments : 1000000;
  for (int a = 0; a < 3; ++a) { R.lo[a] = run->src_lo[a]; R.w[a] = run->src_hi[a] - run->src_lo[a]; }
  R.states = d_states;
  R.out = o->out;
  R.pflags = o->pflags;
  R.pnseg = o->pnseg;
  R.pterm = o->pterm;
  R.trace = o->trace;
  R.trace_cap = trace ? o->trace_cap : 0;
  R.trace_count = reinterpret_cast<unsigned long long*>(o->trace_count);
  R.mesh = m->g.mesh_on ? o->mesh : nullptr;
  R.inst = o->inst;
  R.bank = o->bank;
  R.bank_n = o->bank_n;
  if ((o->bank == nullptr) != (o->bank_n == nullptr))
    return err(NT_E_ARG, std::string(who) + ": outputs.bank and outputs.bank_n go together");
  const unsigned slot = m->slot.fetch_add(1) % kSlots;
  R.counter = m->counters + slot;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaError_t e = cudaMemsetAsync(R.counter, 0, sizeof(unsigned long long), s);
  DevGeom g = m->g;
  if (e == cudaSuccess && dp) {
    // one tracker object per universe, built once per model on its device (vtables of the
    // feature-set module that runs the kernel)
    const bool f0 = m->g.features == 0;
    std::lock_guard<std::mutex> lk(m->dp_mu);
    const size_t ob = f0 ? f0::dp_object_bytes() : f7::dp_object_bytes();
    const size_t nu = (size_t)m->g.n_univ, tab_off = (nu * ob + 255) & ~size_t(255);
    if (!m->dp_objs) {
      e = cudaMalloc(&m->dp_objs, tab_off + nu * sizeof(void*));
      if (e == cudaSuccess) {
        char* base = static_cast<char*>(m->dp_objs);
        e = f0 ? f0::dp_init(m->g, base, base + tab_off, s) : f7::dp_init(m->g, base, base + tab_off, s);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
        if (e != cudaSuccess) { cudaFree(m->dp_objs); m->dp_objs = nullptr; }
      } else {
        m->dp_objs = nullptr;
      }
    }
    if (e == cudaSuccess) g.trk = reinterpret_cast<const void* const*>(static_cast<char*>(m->dp_objs) + tab_off);
  }
  if (e == cudaSuccess && R.bank_n) e = cudaMemsetAsync(R.bank_n, 0, run->n, s);   // F1: no sites by default
  int grid = 0;
  if (e == cudaSuccess) {
    const bool st = d_states != nullptr, f0 = m->g.features == 0;
    if (run->tracker == NT_TRACKER_RECT && (run->flags & NT_HISTORY))
      e = f0::launch_rect(m->g, m->rg, R, trace, st, block, run->blocks_per_sm, s, &grid);
    else if (run->tracker == NT_TRACKER_RECT)
      e = f0r::launch_rect_event(m->g, m->rg, R, trace, st, run->blocks_per_sm, s, &grid);
    else if (run->flags & NT_HISTORY)
      e = f0 ? f0::launch_generic(m->g, R, trace, st, block, run->blocks_per_sm, s, &grid)
             : f7::launch_generic(m->g, R, trace, st, block, run->blocks_per_sm, s, &grid);
    else if (run->flags & NT_WARPQ)
      e = f0 ? f0::launch_wq(m->g, R, trace, st, run->blocks_per_sm, s, &grid)
             : f7::launch_wq(m->g, R, trace, st, run->blocks_per_sm, s, &grid);
    else if (!f0 && async && block == 256 && !trace && !R.mesh && !R.inst && !g.trk &&
             (m->g.features & ~(F_HEX | F_PLANE)) == 0 && !getenv("NESTRACK_NO_FH"))
      e = fh::launch_event_sp(g, R, st, run->blocks_per_sm, s, &grid);   // hex + plane models: smaller kernel
    else
      e = f0 ? f0::launch_event(g, R, trace, st, block, run->blocks_per_sm, s, &grid, async)
             : f7::launch_event(g, R, trace, st, block, run->blocks_per_sm, s, &grid, async);
  }
  if (prev != m->device) cudaSetDevice(prev);
  if (e != cudaSuccess) return cuda_err(e, who);
  m->last_launches = 1;
  return NT_OK;
}

nt_status nt_track(nt_model* m, const nt_run* run, const nt_outputs* o, void* stream) {
  return run_common(m, run, nullptr, o, stream, "nt_track");
}

nt_status nt_track_states(nt_model* m, const nt_run* run, const double* d_states, const nt_outputs* o,
                          void* stream) {
  if (!d_states) return err(NT_E_ARG, "nt_track_states: d_states is NULL");
  return run_common(m, run, d_states, o, stream, "nt_track_states");
}

nt_status nt_track_host(nt_model* m, const nt_run* run, double* host_out, void* stream) {
  if (!m || !run || !host_out) return err(NT_E_ARG, "nt_track_host: NULL argument");
  if (!m->finalized || !m->blob) return err(NT_E_ORDER, "nt_track_host: model not finalized on a device");
  if (run->flags & NT_TRACE) return err(NT_E_ARG, "nt_track_host: tracing needs device buffers");
  std::lock_guard<std::mutex> lk(m->host_mu);
  const size_t len = 2 * (size_t)m->F.n_mc + NT_NC;
  int prev = 0;
  cudaGetDevice(&prev);
  if (prev != m->device) cudaSetDevice(m->device);
  cudaError_t e = cudaSuccess;
  if (m->host_scratch_len < len) {
    if (m->host_scratch_dev) cudaFree(m->host_scratch_dev);
    e = cudaMalloc(&m->host_scratch_dev, len * sizeof(double));
    m->host_scratch_len = e == cudaSuccess ? len : 0;
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (e == cudaSuccess) e = cudaMemsetAsync(m->host_scratch_dev, 0, len * sizeof(double), s);
  if (prev != m->device) cudaSetDevice(prev);
  if (e != cudaSuccess) return cuda_err(e, "nt_track_host");
  nt_outputs o{};
  o.out = m->host_scratch_dev;
  nt_status st = run_common(m, run, nullptr, &o, stream, "nt_track_host");
  if (st != NT_OK) return st;
  if (prev != m->device) cudaSetDevice(m->device);
  e = cudaMemcpyAsync(host_out, m->host_scratch_dev, len * sizeof(double), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (prev != m->device) cudaSetDevice(prev);
  if (e != cudaSuccess) return cuda_err(e, "nt_track_host");
  return NT_OK;
}

nt_status nt_find_cells(nt_model* m, const double* d_xyz, uint64_t n, int32_t* d_cell, uint8_t* d_flag,
                        void* stream) {
  if (!m || (n && (!d_xyz || !d_cell))) return err(NT_E_ARG, "nt_find_cells: NULL argument");
  if (!m->finalized || !m->blob) return err(NT_E_ORDER, "nt_find_cells: model not finalized on a device");
  if (n == 0) return NT_OK;
  int prev = 0;
  cudaGetDevice(&prev);
  if (prev != m->device) cudaSetDevice(m->device);
  cudaError_t e = m->g.features == 0
                      ? f0::launch_find_cells(m->g, d_xyz, n, d_cell, d_flag, static_cast<cudaStream_t>(stream))
                      : f7::launch_find_cells(m->g, d_xyz, n, d_cell, d_flag, static_cast<cudaStream_t>(stream));
  if (prev != m->device) cudaSetDevice(prev);
  if (e != cudaSuccess) return cuda_err(e, "nt_find_cells");
  return NT_OK;
}

int32_t nt_last_launch_count(const nt_model* m) { return m ? m->last_launches : 0; }

// debug (tuning builds with -DNT_BIH_STATS): BIH traversal counters of feature set `fset` (0 / 7)
extern "C" nt_status nt_debug_bih_stats(int32_t fset, uint64_t* out4, int32_t reset) {
  cudaError_t e = fset == 0 ? f0::bih_stats(reinterpret_cast<unsigned long long*>(out4), reset != 0)
                            : f7::bih_stats(reinterpret_cast<unsigned long long*>(out4), reset != 0);
  if (e != cudaSuccess) return cuda_err(e, "nt_debug_bih_stats");
  return NT_OK;
}

// debug: the BIH nodes of CSG universe uid (lmax, rmin, meta, a per node, relative to the root node)
extern "C" nt_status nt_debug_bih_nodes(const nt_model* m, int32_t uid, double* lmax, double* rmin, int32_t* meta,
                                        int32_t* a, int32_t cap, int32_t* n_nodes) {
  if (!m || !m->finalized || uid < 0 || uid >= (int)m->F.univ.size() || m->F.univ[uid].kind != U_CSG)
    return err(NT_E_ARG, "nt_debug_bih_nodes: bad model / universe");
  const int root = m->F.univ[uid].i0;
  int n = 0;
  std::vector<int> todo{root};
  int hi = root;
  while (!todo.empty()) {                      // nodes of this universe: contiguous from root
    const int k = todo.back();
    todo.pop_back();
    hi = std::max(hi, k);
    if (m->F.bih[k].meta >= 0) { todo.push_back(m->F.bih[k].a); todo.push_back(m->F.bih[k].a + 1); }
  }
  for (int k = root; k <= hi; ++k, ++n)
    if (n < cap) {
      const BihNode& b = m->F.bih[k];
      lmax[n] = b.lmax; rmin[n] = b.rmin; meta[n] = b.meta; a[n] = b.meta >= 0 ? b.a - root : b.a;
    }
  *n_nodes = n;
  return NT_OK;
}

nt_status nt_selftest_arith(uint64_t n, uint64_t seed, uint64_t* mismatches) {
  if (!mismatches) return err(NT_E_ARG, "nt_selftest_arith: mismatches is NULL");
  unsigned long long* d = nullptr;
  cudaError_t e = cudaMalloc(&d, 2 * sizeof(unsigned long long));
  if (e == cudaSuccess) e = cudaMemset(d, 0, 2 * sizeof(unsigned long long));
  if (e == cudaSuccess) e = f0::selftest_arith(n, seed, d);
  if (e == cudaSuccess) e = cudaMemcpy(mismatches, d, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
  if (d) cudaFree(d);
  if (e != cudaSuccess) return cuda_err(e, "nt_selftest_arith");
  return NT_OK;
}

}  // extern "C"
