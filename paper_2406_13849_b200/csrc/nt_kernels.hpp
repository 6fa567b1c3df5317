// Kernel launch interface between capi.cpp (host, C++) and the CUDA translation units.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/nestrack.h"
#include "nt_layout.hpp"

namespace nt {

struct KRun {
  uint64_t seed, pid0, n, max_seg;
  double lo[3], w[3];
  const double* states;             // optional SoA [6][n] birth states
  double* out;                      // [len | exits | counters]
  uint8_t* pflags;
  uint32_t* pnseg;
  uint8_t* pterm;
  nt_trace_rec* trace;
  uint64_t trace_cap;
  unsigned long long* trace_count;
  unsigned long long* counter;      // work counter (pid claims), zeroed before launch
  double* slices;                   // [grid][n_mc] zeroed per-block track-length tallies (global)
  double* mesh;                     // optional per-voxel track length (M1), accumulated
  double* inst;                     // optional per-instance track length (D1), accumulated
  double* bank;                     // optional fission sites (F1): [n][max_sites][3]
  uint8_t* bank_n;                  //   sites banked by each history (zeroed by the caller)
};

// one copy of the launchers per compiled feature set (track_f0.cu, track_f7.cu)
#define NT_LAUNCHERS \
cudaError_t upload_coefficients(const double* host, int n); \
cudaError_t launch_generic(const DevGeom& g, const KRun& R, bool trace, bool states, int block, \
                           int blocks_per_sm, cudaStream_t stream, int* grid_out); \
cudaError_t launch_rect(const DevGeom& g, const RectGeom& rg, const KRun& R, bool trace, bool states, \
                        int block, int blocks_per_sm, cudaStream_t stream, int* grid_out); \
cudaError_t launch_event(const DevGeom& g, const KRun& R, bool trace, bool states, int block, \
                         int blocks_per_sm, cudaStream_t stream, int* grid_out, bool async = false); \
cudaError_t launch_wq(const DevGeom& g, const KRun& R, bool trace, bool states, int blocks_per_sm, \
                      cudaStream_t stream, int* grid_out); \
cudaError_t dp_init(const DevGeom& g, void* objs, void* tab, cudaStream_t stream); \
size_t dp_object_bytes(); \
cudaError_t bank_compact(const DevGeom& g, const double* bank, const uint8_t* bank_n, uint64_t n, double* sites, \
                         unsigned long long* M_host, cudaStream_t stream); \
cudaError_t source_from_sites(const double* sites, unsigned long long M, uint64_t seed, uint32_t cycle, \
                              uint64_t j_begin, uint64_t n_next, double* states, cudaStream_t stream); \
cudaError_t fission_source(const DevGeom& g, const double* bank, const uint8_t* bank_n, uint64_t n_prev, \
                           uint64_t seed, uint32_t cycle, uint64_t n_next, double* states, \
                           unsigned long long* M_host, cudaStream_t stream); \
cudaError_t selftest_arith(uint64_t n, uint64_t seed, unsigned long long* d_bad); \
cudaError_t bih_stats(unsigned long long* host4, bool reset); \
cudaError_t launch_find_cells(const DevGeom& g, const double* xyz, uint64_t n, int32_t* cell, \
                              uint8_t* flag, cudaStream_t stream); \

namespace f0 { NT_LAUNCHERS }
namespace f7 { NT_LAUNCHERS }
// track_fh.cu: hex + general-plane models, default path only (own coefficient table)
namespace fh {
cudaError_t upload_coefficients(const double* host, int n);
cudaError_t launch_event_sp(const DevGeom& g, const KRun& R, bool states, int blocks_per_sm, cudaStream_t stream,
                            int* grid_out);
}
// track_rect.cu: the rect-specialised tracker under the ring scheduler (own coefficient table)
namespace f0r {
cudaError_t upload_coefficients(const double* host, int n);
cudaError_t launch_rect_event(const DevGeom& g, const RectGeom& rg, const KRun& R, bool trace, bool states,
                              int blocks_per_sm, cudaStream_t stream, int* grid_out);
}

}  // namespace nt
