// TCGEN05 family: one 128 x BN UMMA tile per CTA, bf16 operands staged by TMA
// into 128-byte-swizzled shared memory, fp32 accumulator in TMEM.
//
// Warp roles (128 threads):
//   warp 0   : TMEM allocation; lane 0 is the TMA producer
//   warp 1   : lane 0 initialises the mbarriers and issues tcgen05.mma
//   warps 2-3: split-K bookkeeping (arrival ticket, zeroing of the tile)
//   warps 0-3: epilogue -- tcgen05.ld of their 32 TMEM lanes (= 32 output
//              rows) into shared memory over the finished ring, then TMA
//              store / add-reduce (BN % 32 == 0) or thread stores / red.add.
// Launched with programmatic dependent launch: setup (TMEM allocation,
// barrier init, descriptor prefetch) overlaps the previous grid's tail and
// griddepcontrol.wait guards every global access.  No cluster attribute:
// a 1x1x1 cluster launch costs 0.06-0.25 us per launch (profiles/r02_gemm_lab.md).
// The k loop is an S-stage smem ring: full[s] (TMA tx-count) and empty[s]
// (tcgen05.commit) mbarriers.
//
// Split-K (plan.hpp tc_geom):
//   mode 0 -- no split: plain (TMA) stores;
//   mode 2 -- right after griddepcontrol.wait, warp 2 takes an arrival ticket
//     per tile (per-candidate counter, never reset within a measure call, so
//     launch L owns tickets [L*splits, (L+1)*splits)); the CTA holding the
//     tile's first ticket of this launch zeroes the tile while its operands
//     stream in and releases a flag (value = launch epoch + 1); every CTA adds
//     its partial after acquiring that flag;
//   mode 3 -- more tiles than ticket slots: fp32 red.add into a C the runner
//     memsets before the launch.
// Instantiated at runtime for any BN in [16, 256] step 16, split-K ways,
// k-tiles and stage count (see plan.cpp).
//
// fp32 workloads (X3): the same tile as 3xTF32 -- see the X3 note at the
// kernel template; cfg[8] = 1 in the planner's report.
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
  int ld;
  uint32_t* sync;             // mode 2: [kTcSyncSlots] tickets, then [kTcSyncSlots] ready flags
  unsigned long long* trace;  // optional per-CTA globaltimer stamps (8 per CTA)
  uint32_t idesc;
  uint32_t tmem_cols;
  int lo_b;  // X3: batch index offset of the lo halves in the operand maps
};

constexpr int kTile = 128 * 64 * 2;  // A stage bytes

// epilogue kinds
constexpr int kEpiStaged = 0;  // padded smem tile, thread float4 stores / red.add (BN % 32 != 0, mode 3)
constexpr int kEpiTma = 1;     // 32-column 128B-swizzled chunks, TMA store / add-reduce
constexpr int kEpiDirect = 2;  // mode 0, BN <= 32: each thread stores its TMEM row from registers

// One instantiation per (split-K mode, epilogue, tracing): every launch runs
// straight-line code for its own case (the all-cases kernel measured 0.5 us
// slower per bmm launch, profiles/r02_gemm_lab.md §5).
//
// X3 (fp32 workloads, 3xTF32): the operands come as [hi | lo] pairs of fp32
// tensors (hi = the top 19 bits, lo = the exact remainder; launch_split_tf32),
// a stage holds one 32-element k sub-tile of A_hi, A_lo, B_hi, B_lo (each
// 128-byte rows, the bf16 stage's layout), and each 8-deep k step issues
// lo*hi + hi*lo + hi*hi as kind::tf32 UMMAs into the fp32 accumulator: fp32
// accuracy (the dropped lo*lo term is ~2^-22 relative) at tensor-core rate.
template <int MODE, int EPI, bool TRACE, bool X3>
__global__ void __launch_bounds__(128, 1)
tc_gemm_kernel(const __grid_constant__ CUtensorMap tma, const __grid_constant__ CUtensorMap tmb,
               const __grid_constant__ CUtensorMap tmc, TcArgs a) {
  static_assert(EPI != kEpiDirect || MODE == 0, "direct epilogue stores: no split");
  extern __shared__ uint8_t smem_raw[];
  __shared__ uint32_t s_ticket;
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* gbase = smem_raw + (base - raw);
  const int b_bytes = a.bn * 64 * 2;            // one operand tile: BN rows of 128 bytes
  constexpr int kHalves = X3 ? 2 : 1;           // X3: hi and lo tiles of each operand
  const uint32_t a0 = base;                     // A stages
  const uint32_t b0 = base + a.stages * kTile * kHalves;  // B stages
  const uint32_t ring = static_cast<uint32_t>(a.stages * (kTile + b_bytes) * kHalves);
  const uint32_t tile_bytes = EPI == kEpiDirect ? 0u
                              : EPI == kEpiTma  ? static_cast<uint32_t>(a.bn / 32) * 16384u
                                                : static_cast<uint32_t>(128 * a.ld * 4);
  const uint32_t bars = (base + (ring > tile_bytes ? ring : tile_bytes) + 15u) & ~15u;
  const uint32_t full = bars, empty = bars + 8 * a.stages, done = bars + 16 * a.stages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(gbase + (done + 8 - base));

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_blk = blockIdx.x, m_blk = blockIdx.y;
  unsigned long long* tr = nullptr;
  if constexpr (TRACE) {
    const size_t cta = (static_cast<size_t>(blockIdx.z) * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
    tr = a.trace + 8 * cta;
    if (threadIdx.x == 0) tr[0] = gtime();
  }
  const int batch = MODE == 0 ? static_cast<int>(blockIdx.z) : static_cast<int>(blockIdx.z) / a.splits;
  const int split = MODE == 0 ? 0 : static_cast<int>(blockIdx.z) % a.splits;

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
  if (TRACE && threadIdx.x == 0) tr[1] = gtime();

  const uint32_t stage_bytes = (kTile + b_bytes) * kHalves;
  const int tile = (batch * gridDim.y + m_blk) * gridDim.x + n_blk;
  float* ctile = a.c + batch * a.sc_b + static_cast<int64_t>(m_blk) * 128 * a.sc_m + static_cast<int64_t>(n_blk) * a.bn;
  const int c4 = a.bn / 4;
  // programmatic dependent launch: this grid waits for its predecessor before
  // its first global access, then lets the next grid start its prologue.
  // Triggering only after the wait keeps at most one grid ahead resident: a
  // trigger before the wait lets a whole chain of waiting grids pile onto the
  // SMs (bmm 2.91 -> 1.84 us per launch in a 2000-launch chain,
  // profiles/r02_gemm_lab.md §5)
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

  if constexpr (MODE == 2) {
    if (warp >= 2) {
      // every CTA takes its arrival ticket now (off the critical path); the
      // first CTA of the tile to start zeroes it while its operands stream in
      const int t2 = threadIdx.x - 64;
      if (t2 == 0) s_ticket = atomicAdd(a.sync + tile, 1u);
      asm volatile("bar.sync 1, 64;" ::: "memory");
      const uint32_t t = s_ticket;
      if (t % static_cast<uint32_t>(a.splits) == 0) {
        const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int e = t2; e < 128 * c4; e += 64) {
          const int r = e / c4, cc = (e % c4) * 4;
          *reinterpret_cast<float4*>(ctile + static_cast<int64_t>(r) * a.sc_m + cc) = z;
        }
        asm volatile("bar.sync 1, 64;" ::: "memory");
        if (t2 == 0) st_release_u32(a.sync + kTcSyncSlots + tile, t / static_cast<uint32_t>(a.splits) + 1);
      }
    }
  }

  if (warp == 0 && lane == 0) {
    // ---- TMA producer ----
    int s = 0;
    uint32_t ph = 0;
    constexpr int kStep = X3 ? 32 : 64;  // k elements per stage (128-byte rows)
    int kc = split * a.kt * kStep;
    for (int kt = 0; kt < a.kt; ++kt, kc += kStep) {
      if (kt >= a.stages) mbar_wait(empty + 8 * s, ph ^ 1);
      mbar_expect_tx(full + 8 * s, stage_bytes);
      tma_load_3d(a0 + s * kTile * kHalves, &tma, full + 8 * s, kc, m_blk * 128, batch);
      tma_load_3d(b0 + s * b_bytes * kHalves, &tmb, full + 8 * s, kc, n_blk * a.bn, batch);
      if constexpr (X3) {
        tma_load_3d(a0 + s * kTile * 2 + kTile, &tma, full + 8 * s, kc, m_blk * 128, batch + a.lo_b);
        tma_load_3d(b0 + s * b_bytes * 2 + b_bytes, &tmb, full + 8 * s, kc, n_blk * a.bn, batch + a.lo_b);
      }
      if (++s == a.stages) {
        s = 0;
        ph ^= 1;
      }
    }
  } else if (warp == 1 && lane == 0) {
    // ---- MMA issuer (single thread) ----
    int s = 0;
    uint32_t ph = 0;
    for (int kt = 0; kt < a.kt; ++kt) {
      mbar_wait(full + 8 * s, ph);
      tc_fence_after();
      if (TRACE && kt == 0) tr[2] = gtime();
      const uint32_t sa = a0 + s * kTile * kHalves, sb = b0 + s * b_bytes * kHalves;
      if constexpr (X3) {
        const uint32_t la = sa + kTile, lb = sb + b_bytes;
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          umma_tf32(tmem, sdesc(la + kk * 32), sdesc(sb + kk * 32), a.idesc, (kt | kk) != 0);
          umma_tf32(tmem, sdesc(sa + kk * 32), sdesc(lb + kk * 32), a.idesc, 1);
          umma_tf32(tmem, sdesc(sa + kk * 32), sdesc(sb + kk * 32), a.idesc, 1);
        }
      } else {
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          umma_bf16(tmem, sdesc(sa + kk * 32), sdesc(sb + kk * 32), a.idesc, (kt | kk) != 0);
      }
      if (kt + a.stages < a.kt) umma_commit(empty + 8 * s);  // the slot is refilled
      if (++s == a.stages) {
        s = 0;
        ph ^= 1;
      }
    }
    umma_commit(done);
  }

  // ---- epilogue ----
  mbar_wait(done, 0);
  __syncwarp();
  tc_fence_after();
  if (TRACE && threadIdx.x == 0) tr[3] = gtime();
  const int row = warp * 32 + lane;  // TMEM lane == output row of this thread
  const uint32_t trow = tmem + (static_cast<uint32_t>(warp * 32) << 16);
  if constexpr (EPI == kEpiDirect) {
    // TMEM -> registers -> the thread's own output row (64-128 contiguous bytes)
    float* dst = ctile + static_cast<int64_t>(row) * a.sc_m;
    for (int c0 = 0; c0 < a.bn; c0 += 16) {
      uint32_t v[16];
      tmem_ld16_nowait(trow + c0, v);
      tmem_wait();
#pragma unroll
      for (int q = 0; q < 4; ++q)
        *reinterpret_cast<float4*>(dst + c0 + 4 * q) =
            make_float4(__uint_as_float(v[4 * q]), __uint_as_float(v[4 * q + 1]), __uint_as_float(v[4 * q + 2]),
                        __uint_as_float(v[4 * q + 3]));
    }
    if (TRACE && threadIdx.x == 0) tr[4] = tr[5] = gtime();
  } else {
    if constexpr (EPI == kEpiTma) {
      // TMEM -> 32-column chunks [128][32] fp32 with the 128-byte swizzle the C
      // tensor map expects (16-byte unit q of row r at q ^ (r & 7): conflict-free)
      for (int c0 = 0; c0 < a.bn; c0 += 32) {
        uint32_t v[32];
        tmem_ld16_nowait(trow + c0, v);
        tmem_ld16_nowait(trow + c0 + 16, v + 16);
        tmem_wait();
        uint8_t* chunk = gbase + (c0 / 32) * 16384 + row * 128;
#pragma unroll
        for (int q = 0; q < 8; ++q)
          *reinterpret_cast<float4*>(chunk + ((q ^ (row & 7)) << 4)) =
              make_float4(__uint_as_float(v[4 * q]), __uint_as_float(v[4 * q + 1]), __uint_as_float(v[4 * q + 2]),
                          __uint_as_float(v[4 * q + 3]));
      }
      fence_proxy_async_smem();  // read by the TMA engine
    } else {
      // TMEM -> padded smem tile over the finished ring (BN = 16 (mod 32))
      float* stg = reinterpret_cast<float*>(gbase) + row * a.ld;
      for (int c0 = 0; c0 < a.bn; c0 += 16) {
        uint32_t v[16];
        tmem_ld16_nowait(trow + c0, v);
        tmem_wait();
#pragma unroll
        for (int q = 0; q < 4; ++q)
          *reinterpret_cast<float4*>(stg + c0 + 4 * q) =
              make_float4(__uint_as_float(v[4 * q]), __uint_as_float(v[4 * q + 1]), __uint_as_float(v[4 * q + 2]),
                          __uint_as_float(v[4 * q + 3]));
      }
    }
    __syncthreads();
    if (TRACE && threadIdx.x == 0) tr[4] = gtime();

    if constexpr (MODE == 2) {
      if (s_ticket % static_cast<uint32_t>(a.splits) != 0) {
        if (threadIdx.x == 0)
          while (ld_acquire_u32(a.sync + kTcSyncSlots + tile) < s_ticket / static_cast<uint32_t>(a.splits) + 1) {
          }
        __syncthreads();
      }
    }
    if (TRACE && threadIdx.x == 0) tr[5] = gtime();
    if constexpr (EPI == kEpiTma) {
      if (threadIdx.x == 0) {
        fence_proxy_async_global();  // the (acquired) zeroing precedes the async-proxy reduction
        for (int c0 = 0; c0 < a.bn; c0 += 32) {
          const uint32_t src = base + (c0 / 32) * 16384;
          if constexpr (MODE == 0) tma_store_3d(&tmc, src, n_blk * a.bn + c0, m_blk * 128, batch);
          else tma_reduce_add_3d(&tmc, src, n_blk * a.bn + c0, m_blk * 128, batch);
        }
        bulk_commit();
        bulk_wait_all();
      }
    } else {
      const float* stile = reinterpret_cast<const float*>(gbase);
      for (int e = threadIdx.x; e < 128 * c4; e += 128) {
        const int r = e / c4, cc = (e % c4) * 4;
        const float4 acc = *reinterpret_cast<const float4*>(stile + r * a.ld + cc);
        float* dst = ctile + static_cast<int64_t>(r) * a.sc_m + cc;
        if constexpr (MODE == 0) *reinterpret_cast<float4*>(dst) = acc;
        else red_add_f4(dst, acc);
      }
    }
  }
  if (TRACE && threadIdx.x == 0) {
    tr[6] = gtime();
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    tr[7] = smid;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(a.tmem_cols) : "memory");
  }
}

using TcKernel = void (*)(CUtensorMap, CUtensorMap, CUtensorMap, TcArgs);

// the instantiations: (mode, epilogue) pairs tc_geom can produce, x tracing x operand kind
template <bool TRACE, bool X3>
TcKernel pick_kernel(int mode, int epi) {
  if (mode == 0) {
    if (epi == kEpiDirect) return tc_gemm_kernel<0, kEpiDirect, TRACE, X3>;
    if (epi == kEpiTma) return tc_gemm_kernel<0, kEpiTma, TRACE, X3>;
    return tc_gemm_kernel<0, kEpiStaged, TRACE, X3>;
  }
  if (mode == 2)
    return epi == kEpiTma ? tc_gemm_kernel<2, kEpiTma, TRACE, X3> : tc_gemm_kernel<2, kEpiStaged, TRACE, X3>;
  return tc_gemm_kernel<3, kEpiStaged, TRACE, X3>;
}

TcKernel pick_kernel(int mode, int epi, bool trace, bool x3) {
  if (x3) return trace ? pick_kernel<true, true>(mode, epi) : pick_kernel<false, true>(mode, epi);
  return trace ? pick_kernel<true, false>(mode, epi) : pick_kernel<false, false>(mode, epi);
}

TcKernel kernel_for(const TcGeom& g, bool trace, bool x3) {
  const int epi = g.direct ? kEpiDirect : g.tma_epi ? kEpiTma : kEpiStaged;
  return pick_kernel(g.mode, epi, trace, x3);
}

// the smem opt-in of every instantiation (identical static smem), once
int tc_max_dyn() {
  static int max_dyn = [] {
    int m = 1 << 30;
    for (int mode : {0, 2, 3})
      for (int epi : {kEpiStaged, kEpiTma, kEpiDirect})
        for (bool t : {false, true})
          for (bool x3 : {false, true}) {
            if (epi == kEpiDirect && mode != 0) continue;
            if (mode == 3 && epi != kEpiStaged) continue;
            const int d = opt_in_dynamic_smem(reinterpret_cast<const void*>(pick_kernel(mode, epi, t, x3)));
            m = std::min(m, d);
          }
    return m;
  }();
  return max_dyn;
}

}  // namespace

void preload_tc_gemm() { tc_max_dyn(); }

bool launch_tc_gemm(const TcLaunch& L, cudaStream_t st) {
  const int max_dyn = tc_max_dyn();
  if (max_dyn <= 0 || L.smem_bytes > max_dyn) return false;
  const TcGeom g = tc_geom(L.bn, L.splits, L.stages, static_cast<int64_t>(L.batch) * L.grid_m * L.grid_n, L.x3);
  if (g.mode == 2 && !L.sync) return false;
  if (g.tma_epi && !L.tmap_c) return false;  // smem was planned for the TMA epilogue
  TcArgs a;
  a.c = L.c;
  a.sc_b = L.sc_b;
  a.sc_m = L.sc_m;
  a.bn = L.bn;
  a.splits = L.splits;
  a.kt = L.x3 ? 2 * L.kt : L.kt;  // X3: stages are 32-element k sub-tiles
  a.lo_b = L.x3 ? L.batch : 0;
  a.stages = L.stages;
  a.ld = g.ld;
  a.sync = L.sync;
  a.trace = L.trace;
  // instruction descriptor: D f32, A/B bf16 (kind::f16) or tf32 (kind::tf32),
  // both K-major, N>>3, M>>4
  const uint32_t fmt = L.x3 ? 2u : 1u;
  a.idesc = (1u << 4) | (fmt << 7) | (fmt << 10) | (static_cast<uint32_t>(L.bn >> 3) << 17) |
            (static_cast<uint32_t>(128 >> 4) << 24);
  uint32_t cols = 32;
  while (cols < static_cast<uint32_t>(L.bn)) cols <<= 1;
  a.tmem_cols = cols;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(L.grid_n), static_cast<unsigned>(L.grid_m),
                     static_cast<unsigned>(L.batch * L.splits));
  cfg.blockDim = dim3(128, 1, 1);
  cfg.dynamicSmemBytes = static_cast<size_t>(L.smem_bytes);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = L.pdl ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const CUtensorMap ta = *static_cast<const CUtensorMap*>(L.tmap_a);
  const CUtensorMap tb = *static_cast<const CUtensorMap*>(L.tmap_b);
  const CUtensorMap tc = L.tmap_c ? *static_cast<const CUtensorMap*>(L.tmap_c) : tb;
  if (cudaLaunchKernelEx(&cfg, kernel_for(g, L.trace != nullptr, L.x3), ta, tb, tc, a) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return cudaGetLastError() == cudaSuccess;
}

}  // namespace lsb
