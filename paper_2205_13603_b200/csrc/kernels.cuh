// Runner kernel launchers (generic families + utilities).  See kernels.cu and
// tc_gemm.cu.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "plan.hpp"

namespace lsb {

// Strides (elements) of the three contraction operands per role.
struct Strides {
  int64_t sx[4], sy[4], sc[4];
  int64_t ext[4];  // batch, m, n, k
};

// Reference output in float64 (one thread per output element).
void launch_reference(const void* x, const void* y, double* out, const Strides& s, bool bf16, cudaStream_t st);
// NAIVE family: one thread per output, fp32 accumulate.
void launch_naive(const void* x, const void* y, float* c, const Strides& s, bool bf16, cudaStream_t st);
// SIMT family (register-tile lattice).
bool launch_simt(const void* x, const void* y, float* c, const Strides& s, const SimtCfg& cfg, bool bf16,
                 const unsigned long long* deadline, int* timed_out, cudaStream_t st);
// LOOPNEST family.
void launch_loopnest(const void* x, const void* y, float* c, const LoopNestCfg& cfg, bool bf16,
                     const unsigned long long* deadline, int* timed_out, cudaStream_t st);
// K6 parity reducer: slot[0] = max |c - ref| (as double bits), slot[1] =
// mismatches; with poison, every checked element is then overwritten with NaN
// so a later candidate that skips an element fails its own check.
void launch_parity(float* c, const double* ref, int64_t n, double rtol, double atol, unsigned long long* slot,
                   bool poison, cudaStream_t st);
// Device-side deadline state: [0] deadline, [1] arm time, [2] best elapsed ns,
// [3] end stamp of the last candidate, [4] calibrated empty-candidate ns.
// arm: first settles the previous candidate (its elapsed time updates best
// when it neither timed out nor failed parity), then sets deadline = now +
// clamp(factor * best, floor, cap) (cap while nothing has succeeded yet).
void launch_arm(unsigned long long* state, const int* prev_flag, const unsigned long long* prev_parity,
                double factor, unsigned long long floor_ns, unsigned long long cap_ns, cudaStream_t st);
// end stamp of a candidate's checked launches: state[3] = now
void launch_stamp(unsigned long long* state, cudaStream_t st);
// spin on the device for ~ns (lets the host queue a chunk of launches)
void launch_delay(unsigned long long ns, cudaStream_t st);
// spins until *flag >= want (mapped pinned host word) or max_ns elapsed
void launch_gate(const unsigned int* flag, unsigned int want, unsigned long long max_ns, cudaStream_t st);
// fp32 -> bf16 copy, and an optional 2-D transpose to make K contiguous
void launch_to_bf16(const float* in, __nv_bfloat16* out, int64_t n, cudaStream_t st);
// 3xTF32 operands of an fp32 contraction: out = [hi | lo] ([2][batch][..]),
// each [batch][cols][rows] (transpose) or [batch][rows][cols] (copy) of in
void launch_split_tf32(const float* in, float* out, int64_t batch, int64_t rows, int64_t cols, bool transpose,
                       cudaStream_t st);
void launch_transpose_bf16(const __nv_bfloat16* in, __nv_bfloat16* out, int64_t batch, int64_t rows,
                           int64_t cols, cudaStream_t st);

// Force-load every runner kernel (CUDA loads functions lazily on first use).
void preload_simt_kernels();
void preload_tc_gemm();
void preload_tc_conv();
void preload_generic_kernels();
// Raise a kernel's dynamic smem limit to the device opt-in minus its static
// smem; returns that limit or -1.
int opt_in_dynamic_smem(const void* fn);

// TCGEN05 family (tc_gemm.cu): tensor maps are built by the caller.
struct TcLaunch {
  const void* tmap_a;  // CUtensorMap* (host memory, passed by value to the kernel)
  const void* tmap_b;
  const void* tmap_c = nullptr;  // fp32 C [batch][M][N], box {32, 128, 1}, 128B swizzle (TMA epilogue)
  float* c;
  int64_t sc_b, sc_m;  // output strides (elements) for batch and M (N contiguous)
  int m, n, k;
  int bn, splits, kt, stages, batch, grid_m, grid_n;
  int smem_bytes;
  unsigned long long* trace = nullptr;  // optional per-CTA timeline (8 stamps per CTA)
  uint32_t* sync = nullptr;             // split-K ticket slots of this candidate (2 x kTcSyncSlots, zeroed)
  bool pdl = true;                      // programmatic dependent launch
  bool x3 = false;  // fp32 operands as 3xTF32: tmap_a / tmap_b cover [hi | lo] (2 x batch), kt in 64-element tiles
};
bool launch_tc_gemm(const TcLaunch& L, cudaStream_t st);

}  // namespace lsb
