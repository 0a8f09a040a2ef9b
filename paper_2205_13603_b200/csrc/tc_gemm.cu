// TCGEN05 family: one 128 x BN UMMA tile per CTA, bf16 operands staged by TMA
// into 128-byte-swizzled shared memory, fp32 accumulator in TMEM.
//
// Warp roles (128 threads):
//   warp 0  : TMEM allocation; lane 0 is the TMA producer
//   warp 1  : lane 0 initialises the mbarriers and issues tcgen05.mma
//   warps 0-3: epilogue -- tcgen05.ld of their 32 TMEM lanes (= 32 output
//             rows), then plain stores (split-K: fp32 red.global.add).
// The k loop is an S-stage smem ring: full[s] (TMA tx-count) and empty[s]
// (tcgen05.commit) mbarriers.  Instantiated at runtime for any BN in
// [16, 256] step 16, split-K ways, k-tiles and stage count (see plan.cpp).
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "kernels.cuh"

namespace lsb {

namespace {

struct TcArgs {
  float* c;
  int64_t sc_b, sc_m;
  int bn, splits, kt, stages, accumulate;
  uint32_t idesc;
  uint32_t tmem_cols;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}

__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap* map, uint32_t bar, int c0, int c1,
                                            int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(
          dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// UMMA shared-memory descriptor: K-major, 128-byte swizzle, 8-row groups 1024 B apart.
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr & 0x3FFFFu) >> 4);
  d |= static_cast<uint64_t>(1) << 16;            // LBO (unused for swizzled K-major)
  d |= static_cast<uint64_t>(1024 >> 4) << 32;    // SBO
  d |= static_cast<uint64_t>(1) << 46;            // descriptor version (sm_100)
  d |= static_cast<uint64_t>(2) << 61;            // SWIZZLE_128B
  return d;
}

__device__ __forceinline__ void umma_bf16(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}

__device__ __forceinline__ void umma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

constexpr int kTile = 128 * 64 * 2;  // A stage bytes

__global__ void __launch_bounds__(128, 1)
tc_gemm_kernel(const __grid_constant__ CUtensorMap tma, const __grid_constant__ CUtensorMap tmb, TcArgs a) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* gbase = smem_raw + (base - raw);
  const int b_bytes = a.bn * 64 * 2;
  const uint32_t a0 = base;                                  // A stages
  const uint32_t b0 = base + a.stages * kTile;               // B stages
  const uint32_t bars = b0 + a.stages * b_bytes;             // full[S], empty[S], done
  const uint32_t full = bars, empty = bars + 8 * a.stages, done = bars + 16 * a.stages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(gbase + (bars - base) + 16 * a.stages + 8);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_blk = blockIdx.x, m_blk = blockIdx.y;
  const int batch = blockIdx.z / a.splits, split = blockIdx.z % a.splits;

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(a.tmem_cols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (threadIdx.x == 32) {
    for (int s = 0; s < a.stages; ++s) {
      mbar_init(full + 8 * s, 1);
      mbar_init(empty + 8 * s, 1);
    }
    mbar_init(done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tma)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmb)) : "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0 && lane == 0) {
    // ---- TMA producer ----
    const uint32_t stage_bytes = kTile + b_bytes;
    for (int kt = 0; kt < a.kt; ++kt) {
      const int s = kt % a.stages;
      const uint32_t ph = (kt / a.stages) & 1;
      if (kt >= a.stages) mbar_wait(empty + 8 * s, ph ^ 1);
      mbar_expect_tx(full + 8 * s, stage_bytes);
      const int kc = (split * a.kt + kt) * 64;
      tma_load_3d(a0 + s * kTile, &tma, full + 8 * s, kc, m_blk * 128, batch);
      tma_load_3d(b0 + s * b_bytes, &tmb, full + 8 * s, kc, n_blk * a.bn, batch);
    }
  } else if (warp == 1 && lane == 0) {
    // ---- MMA issuer (single thread) ----
    for (int kt = 0; kt < a.kt; ++kt) {
      const int s = kt % a.stages;
      const uint32_t ph = (kt / a.stages) & 1;
      mbar_wait(full + 8 * s, ph);
      tc_fence_after();
      const uint32_t sa = a0 + s * kTile, sb = b0 + s * b_bytes;
#pragma unroll
      for (int kk = 0; kk < 4; ++kk)
        umma_bf16(tmem, sdesc(sa + kk * 32), sdesc(sb + kk * 32), a.idesc, (kt | kk) != 0);
      umma_commit(empty + 8 * s);
    }
    umma_commit(done);
  }

  // ---- epilogue: TMEM -> registers -> global ----
  mbar_wait(done, 0);
  __syncwarp();
  tc_fence_after();
  const int row = m_blk * 128 + warp * 32 + lane;
  float* crow = a.c + batch * a.sc_b + static_cast<int64_t>(row) * a.sc_m + static_cast<int64_t>(n_blk) * a.bn;
  for (int c0 = 0; c0 < a.bn; c0 += 16) {
    float v[16];
    tmem_ld16(tmem + (static_cast<uint32_t>(warp * 32) << 16) + c0, v);
    float4* dst = reinterpret_cast<float4*>(crow + c0);
    if (a.accumulate) {
#pragma unroll
      for (int q = 0; q < 4; ++q) atomicAdd(dst + q, make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]));
    } else {
#pragma unroll
      for (int q = 0; q < 4; ++q) dst[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(a.tmem_cols) : "memory");
  }
}

}  // namespace

bool launch_tc_gemm(const TcLaunch& L, cudaStream_t st) {
  static int max_dyn = -1;
  if (max_dyn < 0) max_dyn = opt_in_dynamic_smem(reinterpret_cast<const void*>(tc_gemm_kernel));
  if (max_dyn <= 0 || L.smem_bytes > max_dyn) return false;
  TcArgs a;
  a.c = L.c;
  a.sc_b = L.sc_b;
  a.sc_m = L.sc_m;
  a.bn = L.bn;
  a.splits = L.splits;
  a.kt = L.kt;
  a.stages = L.stages;
  a.accumulate = L.accumulate;
  // kind::f16 instruction descriptor: D f32, A/B bf16, both K-major, N>>3, M>>4
  a.idesc = (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(L.bn >> 3) << 17) |
            (static_cast<uint32_t>(128 >> 4) << 24);
  uint32_t cols = 32;
  while (cols < static_cast<uint32_t>(L.bn)) cols <<= 1;
  a.tmem_cols = cols;
  dim3 grid(static_cast<unsigned>(L.grid_n), static_cast<unsigned>(L.grid_m),
            static_cast<unsigned>(L.batch * L.splits));
  tc_gemm_kernel<<<grid, 128, L.smem_bytes, st>>>(*static_cast<const CUtensorMap*>(L.tmap_a),
                                                  *static_cast<const CUtensorMap*>(L.tmap_b), a);
  return cudaGetLastError() == cudaSuccess;
}

}  // namespace lsb
