// TCGEN05 implicit-GEMM conv family (tc_conv.cu): see affine.hpp TcConvCfg.
#pragma once

#include <cuda_runtime.h>

#include "affine.hpp"

namespace lsb {

// tmap_x: 4-D bf16 map over the X-side buffer [n][h][w][c], box {64, 8, 8, 1};
// tmap_w: 3-D bf16 map over the K-major weight copy [co][k_flat], box {64, bn, 1}.
// cfg.x3 (fp32, 3xTF32): both maps are fp32 over [hi | lo] halves with 32-wide
// boxes -- X with its image dimension doubled (lo at n + x_images), W with a
// batch dimension of 2.
bool launch_tc_conv(const void* tmap_x, const void* tmap_w, float* c, const TcConvCfg& cfg, bool pdl,
                    cudaStream_t st, unsigned long long* trace = nullptr, uint32_t* sync = nullptr,
                    const void* tmap_c = nullptr, const int64_t* oshape = nullptr, int x_images = 0);

}  // namespace lsb
