// TCGEN05 family: one 128 x BN UMMA tile per CTA, bf16 operands staged by TMA
// into 128-byte-swizzled shared memory, fp32 accumulator in TMEM.
//
// Warp roles (128 threads):
//   warp 0  : TMEM allocation; lane 0 is the TMA producer
//   warp 1  : lane 0 initialises the mbarriers and issues tcgen05.mma
// Launched with programmatic dependent launch: setup (TMEM allocation,
// barrier init, descriptor prefetch) overlaps the previous grid's tail and
// griddepcontrol.wait guards every global access.
//   warps 0-3: epilogue -- tcgen05.ld of their 32 TMEM lanes (= 32 output
//             rows) into a shared-memory tile, then coalesced row-segment
//             stores.
// Split-K: the split CTAs of one output tile form a thread-block cluster
// (cluster dims 1 x 1 x splits, <= 16) and reduce their partial tiles through
// distributed shared memory -- each CTA sums one slice of rows across all
// peers (ld.shared::cluster) and writes it once.  No memset, no atomics.
// Above 16 ways the tile falls back to fp32 red.global.add into a zeroed C.
// The k loop is an S-stage smem ring: full[s] (TMA tx-count) and empty[s]
// (tcgen05.commit) mbarriers.  Instantiated at runtime for any BN in
// [16, 256] step 16, split-K ways, k-tiles and stage count (see plan.cpp).
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "kernels.cuh"
#include "tc_common.cuh"

namespace lsb {

namespace {

using namespace tc;

struct TcArgs {
  float* c;
  int64_t sc_b, sc_m;
  int bn, splits, kt, stages;
  int mode;  // 0 single CTA per tile, 1 cluster DSMEM reduction, 2 atomic accumulation
  unsigned long long* trace;  // optional per-CTA globaltimer stamps (8 per CTA)
  uint32_t idesc;
  uint32_t tmem_cols;
};

constexpr int kTile = 128 * 64 * 2;  // A stage bytes
constexpr int kMaxClusterSplits = 16;

__global__ void __launch_bounds__(128, 1)
tc_gemm_kernel(const __grid_constant__ CUtensorMap tma, const __grid_constant__ CUtensorMap tmb, TcArgs a) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* gbase = smem_raw + (base - raw);
  const int b_bytes = a.bn * 64 * 2;
  const uint32_t a0 = base;                                  // A stages
  const uint32_t b0 = base + a.stages * kTile;               // B stages
  const int red_ld = a.bn + 4;                               // padded row (floats)
  const uint32_t stage_end = b0 + a.stages * b_bytes;
  // epilogue buffer: cluster mode receives every peer's rows of this CTA's
  // slice in a region of its own (peers may push while we still run the
  // main loop); single-CTA modes stage their own tile over the finished ring
  const int S_cl = a.mode == 1 ? a.splits : 1;
  const int rows_per = (128 + S_cl - 1) / S_cl;
  const uint32_t red = a.mode == 1 ? ((stage_end + 15u) & ~15u) : base;
  const uint32_t red_bytes = a.mode == 1 ? static_cast<uint32_t>(S_cl * rows_per * red_ld * 4)
                                         : static_cast<uint32_t>(128 * red_ld * 4);
  const uint32_t red_end = red + red_bytes;
  const uint32_t bars = ((stage_end > red_end ? stage_end : red_end) + 15u) & ~15u;
  const uint32_t full = bars, empty = bars + 8 * a.stages, done = bars + 16 * a.stages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(gbase + (bars - base) + 16 * a.stages + 8);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_blk = blockIdx.x, m_blk = blockIdx.y;
  const size_t cta = (static_cast<size_t>(blockIdx.z) * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
  unsigned long long* tr = a.trace ? a.trace + 8 * cta : nullptr;
  if (tr && threadIdx.x == 0) tr[0] = gtime();
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
  if (tr && threadIdx.x == 0) tr[1] = gtime();

  // programmatic dependent launch: the next grid may start its prologue now;
  // this grid waits for its predecessor before its first global access
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");

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
      if (tr && kt == 0) tr[2] = gtime();
      const uint32_t sa = a0 + s * kTile, sb = b0 + s * b_bytes;
#pragma unroll
      for (int kk = 0; kk < 4; ++kk)
        umma_bf16(tmem, sdesc(sa + kk * 32), sdesc(sb + kk * 32), a.idesc, (kt | kk) != 0);
      umma_commit(empty + 8 * s);
    }
    umma_commit(done);
  }

  // ---- epilogue ----
  mbar_wait(done, 0);
  __syncwarp();
  tc_fence_after();
  if (tr && threadIdx.x == 0) tr[3] = gtime();
  const int row = warp * 32 + lane;  // TMEM lane == output row of this thread
  const int c4 = a.bn / 4;
  float* ctile = a.c + batch * a.sc_b + static_cast<int64_t>(m_blk) * 128 * a.sc_m + static_cast<int64_t>(n_blk) * a.bn;
  if (a.mode == 1) {
    // push: row -> the peer that owns its slice, straight from registers
    const uint32_t me = cluster_rank();
    const int owner = row / rows_per, lr = row - owner * rows_per;
    const uint32_t dst =
        map_peer(red + static_cast<uint32_t>(((static_cast<int>(me) * rows_per + lr) * red_ld) * 4), owner);
    for (int c0 = 0; c0 < a.bn; c0 += 16) {
      float v[16];
      tmem_ld16(tmem + (static_cast<uint32_t>(warp * 32) << 16) + c0, v);
#pragma unroll
      for (int q = 0; q < 4; ++q)
        st_cluster_f4(dst + static_cast<uint32_t>((c0 + 4 * q) * 4), v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
    }
    cluster_sync_all();  // every pushed row has landed
    if (tr && threadIdx.x == 0) tr[4] = gtime();
    const int r_lo = static_cast<int>(me) * rows_per;
    const int nrows = min(128, r_lo + rows_per) - r_lo;
    const float* rb = reinterpret_cast<const float*>(gbase + (red - base));
    for (int e = threadIdx.x; e < nrows * c4; e += 128) {
      const int lr2 = e / c4, cc = (e % c4) * 4;
      float4 v[kMaxClusterSplits];
#pragma unroll
      for (int q = 0; q < kMaxClusterSplits; ++q)
        if (q < S_cl) v[q] = *reinterpret_cast<const float4*>(rb + (q * rows_per + lr2) * red_ld + cc);
      float4 acc = v[0];
#pragma unroll
      for (int q = 1; q < kMaxClusterSplits; ++q)
        if (q < S_cl) { acc.x += v[q].x; acc.y += v[q].y; acc.z += v[q].z; acc.w += v[q].w; }
      *reinterpret_cast<float4*>(ctile + static_cast<int64_t>(r_lo + lr2) * a.sc_m + cc) = acc;
    }
  } else {
    // stage the tile over the finished smem ring, then coalesced row segments
    float* stg = reinterpret_cast<float*>(gbase) + row * red_ld;
    for (int c0 = 0; c0 < a.bn; c0 += 16) {
      float v[16];
      tmem_ld16(tmem + (static_cast<uint32_t>(warp * 32) << 16) + c0, v);
#pragma unroll
      for (int q = 0; q < 4; ++q)
        *reinterpret_cast<float4*>(stg + c0 + 4 * q) = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
    }
    __syncthreads();
    if (tr && threadIdx.x == 0) tr[4] = gtime();
    const float* sb = reinterpret_cast<const float*>(gbase);
    for (int e = threadIdx.x; e < 128 * c4; e += 128) {
      const int r = e / c4, cc = (e % c4) * 4;
      const float4 acc = *reinterpret_cast<const float4*>(sb + r * red_ld + cc);
      float4* dst = reinterpret_cast<float4*>(ctile + static_cast<int64_t>(r) * a.sc_m + cc);
      if (a.mode == 2) atomicAdd(dst, acc);
      else *dst = acc;
    }
  }
  if (tr && threadIdx.x == 0) {
    tr[5] = gtime();
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    tr[6] = smid;
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
  a.mode = L.splits == 1 ? 0 : (L.splits <= kMaxClusterSplits ? 1 : 2);
  a.trace = L.trace;
  // kind::f16 instruction descriptor: D f32, A/B bf16, both K-major, N>>3, M>>4
  a.idesc = (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(L.bn >> 3) << 17) |
            (static_cast<uint32_t>(128 >> 4) << 24);
  uint32_t cols = 32;
  while (cols < static_cast<uint32_t>(L.bn)) cols <<= 1;
  a.tmem_cols = cols;
  static bool nonportable = false;
  if (a.mode == 1 && L.splits > 8 && !nonportable) {
    if (cudaFuncSetAttribute(tc_gemm_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess) {
      cudaGetLastError();
      return false;
    }
    nonportable = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(L.grid_n), static_cast<unsigned>(L.grid_m),
                     static_cast<unsigned>(L.batch * L.splits));
  cfg.blockDim = dim3(128, 1, 1);
  cfg.dynamicSmemBytes = static_cast<size_t>(L.smem_bytes);
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 1;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = a.mode == 1 ? static_cast<unsigned>(L.splits) : 1u;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = L.pdl ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  const CUtensorMap ta = *static_cast<const CUtensorMap*>(L.tmap_a);
  const CUtensorMap tb = *static_cast<const CUtensorMap*>(L.tmap_b);
  if (cudaLaunchKernelEx(&cfg, tc_gemm_kernel, ta, tb, a) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return cudaGetLastError() == cudaSuccess;
}

}  // namespace lsb
