// SIMT-A launcher interface.  See simta_impl.cuh / affine.hpp.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "affine.hpp"

namespace lsb {

// One level-list of parts (nest order): extents and per-part address
// coefficients in X, Y, C and the two guarded X dims.
struct AList {
  int n;
  int64_t ext[8], cx[8], cy[8], cc[8], cg0[8], cg1[8];
};

struct SimtaArgs {
  AList m_grid, n_grid, m_thr, n_thr, m_reg, n_reg, k_tile, k_bk;
  int64_t x0, y0, c0;
  int ng;
  int64_t g0[2], gext[2];
  int64_t gm, gn, tm, tn, bk, kt;
  const unsigned long long* deadline;
  int* timed_out;
  int persist;              // checked launches: one wave loops over the tiles (fast timeouts, see kernels.cu)
  int64_t ntn, ntm;         // tile counts of the plain grid (x, y)
};

int opt_in_dynamic_smem(const void* fn);
void preload_simta_f32();
void preload_simta_bf16();
bool launch_simta(const void* x, const void* y, float* c, const AffineCfg& A, bool bf16,
                  const unsigned long long* deadline, int* timed_out, cudaStream_t st);
cudaError_t launch_simta_f32(const void* x, const void* y, float* c, const SimtaArgs& a, int rm, int rn, size_t smem,
                             cudaStream_t st);
cudaError_t launch_simta_bf16(const void* x, const void* y, float* c, const SimtaArgs& a, int rm, int rn, size_t smem,
                              cudaStream_t st);

}  // namespace lsb
