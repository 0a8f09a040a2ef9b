// TCGEN05 implicit-GEMM convolution (NHWC): one CTA owns an 8 x 8 box of
// output pixels x BN output channels.  Each k-tile is one (filter tap, 64
// input channels) pair: TMA loads the 8 x 8 x 64 input box at the tap's shifted
// coordinates straight from the (unpadded or padded) activation tensor into
// the upper 64 rows of a 128-row, 128-byte-swizzled operand stage -- the
// zero padding of the convolution is TMA's out-of-bounds fill, so an inlined
// pad stage costs nothing -- and the matching [BN x 64] slice of the K-major
// weight copy.  The lower 64 rows are dead (never written, never read back):
// the UMMA tile is 128 x BN with half its rows live (M = 64 output pixels
// per box) -- unless the CTA takes a PAIR of boxes (`pair`, split-K modes 0
// and 2; BN 16 tiles or grids above two CTAs per SM): box 2j in rows 0..63 and box
// 2j+1 in rows 64..127 of every stage, one weight slice for both, so every
// UMMA row is live and the grid halves.
//
// Warp roles and pipeline as in tc_gemm.cu (TMA producer lane, single MMA
// issuer, S-stage mbarrier ring, PDL).  Filter-row parts hoisted above every
// spatial loop are split-K: the split CTAs form a cluster and reduce through
// DSMEM (each CTA owns a slice of the 64 live rows).  Coordinates of every
// box come from per-part contributions computed by the planner
// (affine.cpp tc_conv_plan), so any loop order of the scheduled nest maps to
// the same kernel.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include <algorithm>

#include "kernels.cuh"
#include "tc_common.cuh"
#include "tc_conv.cuh"

namespace lsb {

namespace {

using namespace tc;

constexpr int kStageA = 128 * 64 * 2;  // A stage bytes (rows 64..127 zero)
constexpr int kLiveA = 64 * 64 * 2;    // bytes TMA writes per A stage
constexpr int kRows = 64;
constexpr int kMaxClusterSplits = 16;

// X-box / weight-K coordinates of one (split, k-tile) pair, relative to the
// CTA origin; precomputed on the host so the TMA producer does one table
// lookup per k-tile (the mixed-radix decode of the k parts used to cost the
// single producer thread ~1000 cycles of 64-bit division per k-tile).
struct KCoord {
  int32_t c, w, h, n, kf, pad;
};

struct TcConvArgs {
  float* c;
  CList m_grid, n_grid;       // origin parts of the output-pixel box and channel tile
  int64_t x_n0, x_h0, x_w0, x_c0, c0, cc_h1, cc_w1;
  KCoord kc[kConvMaxK];       // [split * kt + k-tile]
  int bn, splits, kt, stages, mode;
  uint32_t idesc, tmem_cols;
  unsigned long long* trace;  // optional per-CTA globaltimer stamps (8 per CTA, as tc_gemm)
  uint32_t* sync;             // mode 2: [kTcSyncSlots] tickets + [kTcSyncSlots] zeroing flags per tile
  int tma_epi;                // modes 0/2: 128B-swizzled [64 px][32 ch] chunks -> 4-D TMA store / add-reduce
  int pair;                   // two boxes per CTA (grid y = pairs of boxes)
  int grid_m;                 // boxes (pair: the odd last pair has one)
  int64_t oshape[4];          // output [n][p][q][k] (decodes the box origin for the C tensor map)
  int lo_n;                   // X3: image offset of the lo halves in the X map
};

struct Coord {
  int64_t n, h, w, c, kf, co, cc;
};

// origin decode: 32-bit mixed radix (grid indices and extents fit in int32)
__device__ __forceinline__ void add_parts(const CList& L, uint32_t idx, Coord& a) {
  for (int i = L.n - 1; i >= 0; --i) {
    const uint32_t e = static_cast<uint32_t>(L.ext[i]);
    const uint32_t q = idx / e;
    const int64_t v = static_cast<int64_t>(idx - q * e);
    idx = q;
    a.n += v * L.xn[i];
    a.h += v * L.xh[i];
    a.w += v * L.xw[i];
    a.c += v * L.xc[i];
    a.kf += v * L.kf[i];
    a.co += v * L.co[i];
    a.cc += v * L.cc[i];
  }
}

void host_add_parts(const CList& L, int64_t idx, Coord& a) {
  for (int i = L.n - 1; i >= 0; --i) {
    const int64_t v = idx % L.ext[i];
    idx /= L.ext[i];
    a.n += v * L.xn[i];
    a.h += v * L.xh[i];
    a.w += v * L.xw[i];
    a.c += v * L.xc[i];
    a.kf += v * L.kf[i];
    a.co += v * L.co[i];
    a.cc += v * L.cc[i];
  }
}

// one instantiation per (split-K mode, epilogue, tracing, operand kind), as
// tc_gemm.cu.  X3 (fp32 workloads, 3xTF32): a ring slot holds one 32-channel
// k sub-tile -- A_hi, A_lo, B_hi, B_lo, each in the bf16 slot's 128-byte-row
// layout -- two slots per (tap, 64 channels) k-tile, and each 8-deep k step
// issues lo*hi + hi*lo + hi*hi as kind::tf32 UMMAs (tc_gemm.cu X3).
template <int MODE, bool TMA_EPI, bool TRACE, bool X3>
__global__ void __launch_bounds__(128, 1)
tc_conv_kernel(const __grid_constant__ CUtensorMap tmx, const __grid_constant__ CUtensorMap tmw,
               const __grid_constant__ CUtensorMap tmc, const __grid_constant__ TcConvArgs a) {
  static_assert(!(TMA_EPI && MODE == 1), "the cluster reduction stores from registers");
  static_assert(!(X3 && MODE == 1), "3xTF32: L2 split-K only");
  constexpr int kH = X3 ? 2 : 1;  // operand halves per slot
  extern __shared__ uint8_t smem_raw[];
  __shared__ uint32_t s_ticket;
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* gbase = smem_raw + (base - raw);
  const int b_bytes = a.bn * 64 * 2;
  const uint32_t a0 = base;
  const uint32_t b0 = base + a.stages * kStageA * kH;
  const int red_ld = a.bn + 4;
  const uint32_t stage_end = b0 + a.stages * b_bytes * kH;
  const int S_cl = MODE == 1 ? a.splits : 1;
  const int rows_per = (kRows + S_cl - 1) / S_cl;
  const uint32_t red = MODE == 1 ? ((stage_end + 15u) & ~15u) : base;
  const uint32_t red_bytes = MODE == 1 ? static_cast<uint32_t>(S_cl * rows_per * red_ld * 4)
                                       : static_cast<uint32_t>((a.pair ? 2 : 1) * kRows * red_ld * 4);
  const uint32_t red_end = red + red_bytes;
  const uint32_t bars = ((stage_end > red_end ? stage_end : red_end) + 15u) & ~15u;
  const uint32_t full = bars, empty = bars + 8 * a.stages, done = bars + 16 * a.stages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(gbase + (bars - base) + 16 * a.stages + 8);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned long long* tr = nullptr;
  if constexpr (TRACE) {
    const size_t cta = (static_cast<size_t>(blockIdx.z) * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
    tr = a.trace + 8 * cta;
    if (threadIdx.x == 0) tr[0] = gtime();
  }

  // The dead lower half of every A stage (rows 64..127) is left as it is:
  // row r of the accumulator depends on A row r only, and rows 64..127 are
  // never read back, so whatever the smem holds there cannot reach C
  // (zeroing it cost ~0.5 us of every CTA's setup).

  // this split's k-tile coordinate table, param space -> smem before the
  // dependency wait (dynamically indexed param reads miss the constant cache
  // on the producer's critical path)
  __shared__ KCoord s_kc[kConvMaxK];
  for (int i = static_cast<int>(threadIdx.x) - 64; i >= 0 && i < a.kt; i += 64) s_kc[i] = a.kc[blockIdx.z * a.kt + i];

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
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmx)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmw)) : "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (TRACE && threadIdx.x == 0) tr[1] = gtime();

  // tile origin: output-pixel box (grid y; a pair of boxes with `pair`),
  // channel tile (grid x), split (grid z)
  const uint32_t box0 = a.pair ? 2u * blockIdx.y : blockIdx.y;
  const int nbox = a.pair && static_cast<int>(box0) + 1 < a.grid_m ? 2 : 1;
  Coord o{a.x_n0, a.x_h0, a.x_w0, a.x_c0, 0, 0, a.c0};
  add_parts(a.m_grid, box0, o);
  add_parts(a.n_grid, blockIdx.x, o);
  Coord o1 = o;
  if (nbox == 2) {
    o1 = Coord{a.x_n0, a.x_h0, a.x_w0, a.x_c0, 0, 0, a.c0};
    add_parts(a.m_grid, box0 + 1, o1);
    add_parts(a.n_grid, blockIdx.x, o1);
  }
  const KCoord* kc = s_kc;

  asm volatile("griddepcontrol.wait;" ::: "memory");  // trigger after the wait: see tc_gemm.cu
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int tile = blockIdx.y * gridDim.x + blockIdx.x;
  const int live = nbox * kRows;  // accumulator rows that hold output pixels
  // row r (0..live-1): box r / 64, pixel r % 64 of that box
  auto out_row = [&](int r) {
    float* cb = a.c + (r >= kRows ? o1.cc : o.cc);
    r &= kRows - 1;
    return cb + (r >> 3) * a.cc_h1 + (r & 7) * a.cc_w1;
  };
  const int c4 = a.bn / 4;
  if (MODE == 2 && warp >= 2) {
    // split-K through L2 (as tc_gemm.cu mode 2): arrival ticket per tile; the
    // first CTA of the tile to start zeroes its 64 x BN output box while its
    // operands stream in and releases this launch's epoch
    const int t2 = threadIdx.x - 64;
    if (t2 == 0) s_ticket = atomicAdd(a.sync + tile, 1u);
    asm volatile("bar.sync 1, 64;" ::: "memory");
    const uint32_t t = s_ticket;
    if (t % static_cast<uint32_t>(a.splits) == 0) {
      const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int e = t2; e < live * c4; e += 64) {
        const int r = e / c4, cc = (e % c4) * 4;
        *reinterpret_cast<float4*>(out_row(r) + cc) = z;
      }
      asm volatile("bar.sync 1, 64;" ::: "memory");
      if (t2 == 0) st_release_u32(a.sync + kTcSyncSlots + tile, t / static_cast<uint32_t>(a.splits) + 1);
    }
  }

  if (warp == 0 && lane == 0) {
    // ---- TMA producer ----
    const uint32_t stage_bytes = (nbox * kLiveA + b_bytes) * kH;
    int s = 0;
    uint32_t ph = 0;
    for (int kt = 0; kt < a.kt * kH; ++kt) {
      if (kt >= a.stages) mbar_wait(empty + 8 * s, ph ^ 1);
      const KCoord k = kc[X3 ? kt >> 1 : kt];
      const int sub = X3 ? 32 * (kt & 1) : 0;  // X3: channel offset of the 32-wide sub-tile
      mbar_expect_tx(full + 8 * s, stage_bytes);
      tma_load_4d(a0 + s * kStageA * kH, &tmx, full + 8 * s, static_cast<int>(o.c) + k.c + sub,
                  static_cast<int>(o.w) + k.w, static_cast<int>(o.h) + k.h, static_cast<int>(o.n) + k.n);
      if constexpr (X3) {
        tma_load_4d(a0 + s * kStageA * 2 + kStageA, &tmx, full + 8 * s, static_cast<int>(o.c) + k.c + sub,
                    static_cast<int>(o.w) + k.w, static_cast<int>(o.h) + k.h, static_cast<int>(o.n) + k.n + a.lo_n);
        tma_load_3d(b0 + s * b_bytes * 2, &tmw, full + 8 * s, static_cast<int>(o.kf) + k.kf + sub,
                    static_cast<int>(o.co), 0);
        tma_load_3d(b0 + s * b_bytes * 2 + b_bytes, &tmw, full + 8 * s, static_cast<int>(o.kf) + k.kf + sub,
                    static_cast<int>(o.co), 1);
        if (++s == a.stages) {
          s = 0;
          ph ^= 1;
        }
        continue;
      }
      if (nbox == 2)  // rows 64..127: the second box (8 KB = 8 swizzle atoms in)
        tma_load_4d(a0 + s * kStageA + kLiveA, &tmx, full + 8 * s, static_cast<int>(o1.c) + k.c,
                    static_cast<int>(o1.w) + k.w, static_cast<int>(o1.h) + k.h, static_cast<int>(o1.n) + k.n);
      tma_load_3d(b0 + s * b_bytes, &tmw, full + 8 * s, static_cast<int>(o.kf) + k.kf, static_cast<int>(o.co), 0);
      if (++s == a.stages) {
        s = 0;
        ph ^= 1;
      }
    }
  } else if (warp == 1 && lane == 0) {
    // ---- MMA issuer (single thread) ----
    int s = 0;
    uint32_t ph = 0;
    for (int kt = 0; kt < a.kt * kH; ++kt) {
      mbar_wait(full + 8 * s, ph);
      tc_fence_after();
      if (TRACE && kt == 0) tr[2] = gtime();
      const uint32_t sa = a0 + s * kStageA * kH, sb = b0 + s * b_bytes * kH;
      if constexpr (X3) {
        const uint32_t la = sa + kStageA, lb = sb + b_bytes;
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
      umma_commit(empty + 8 * s);
      if (++s == a.stages) {
        s = 0;
        ph ^= 1;
      }
    }
    umma_commit(done);
  }

  // ---- epilogue: rows 0..live-1 (TMEM lanes of warps 0-1, and 2-3 for a pair) ----
  mbar_wait(done, 0);
  __syncwarp();
  tc_fence_after();
  if (TRACE && threadIdx.x == 0) tr[3] = gtime();
  const int row = warp * 32 + lane;
  if constexpr (MODE == 1) {
    const uint32_t me = cluster_rank();
    if (warp < 2) {
      const int owner = row / rows_per, lr = row - owner * rows_per;
      const uint32_t dst =
          map_peer(red + static_cast<uint32_t>(((static_cast<int>(me) * rows_per + lr) * red_ld) * 4), owner);
      for (int c0 = 0; c0 < a.bn; c0 += 16) {
        float v[16];
        tmem_ld16(tmem + (static_cast<uint32_t>(warp * 32) << 16) + c0, v);
#pragma unroll
        for (int q = 0; q < 4; ++q)
          st_cluster_f4(dst + static_cast<uint32_t>((c0 + 4 * q) * 4), v[4 * q], v[4 * q + 1], v[4 * q + 2],
                        v[4 * q + 3]);
      }
    }
    cluster_sync_all();
    const int r_lo = static_cast<int>(me) * rows_per;
    const int nrows = max(0, min(kRows, r_lo + rows_per) - r_lo);
    const float* rb = reinterpret_cast<const float*>(gbase + (red - base));
    for (int e = threadIdx.x; e < nrows * c4; e += 128) {
      const int lr2 = e / c4, cc = (e % c4) * 4;
      float4 acc = *reinterpret_cast<const float4*>(rb + lr2 * red_ld + cc);
#pragma unroll
      for (int q = 1; q < kMaxClusterSplits; ++q)
        if (q < S_cl) {
          const float4 v = *reinterpret_cast<const float4*>(rb + (q * rows_per + lr2) * red_ld + cc);
          acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
        }
      *reinterpret_cast<float4*>(out_row(r_lo + lr2) + cc) = acc;
    }
  } else if constexpr (TMA_EPI) {
    // TMEM rows -> per box [64 px][32 ch] fp32 chunks, 128-byte swizzle (unit
    // q of row r at q ^ (r & 7)), then one 4-D TMA store / add-reduce per chunk
    const int nch = a.bn / 32;
    if (row < live) {
      const uint32_t trow = tmem + (static_cast<uint32_t>(warp * 32) << 16);
      for (int c0 = 0; c0 < a.bn; c0 += 32) {
        uint32_t v[32];
        tmem_ld16_nowait(trow + c0, v);
        tmem_ld16_nowait(trow + c0 + 16, v + 16);
        tmem_wait();
        uint8_t* chunk = gbase + ((row >> 6) * nch + c0 / 32) * 8192 + (row & 63) * 128;
#pragma unroll
        for (int q = 0; q < 8; ++q)
          *reinterpret_cast<float4*>(chunk + ((q ^ (row & 7)) << 4)) =
              make_float4(__uint_as_float(v[4 * q]), __uint_as_float(v[4 * q + 1]), __uint_as_float(v[4 * q + 2]),
                          __uint_as_float(v[4 * q + 3]));
      }
    }
    fence_proxy_async_smem();
    __syncthreads();
    if (TRACE && threadIdx.x == 0) tr[4] = gtime();
    if (MODE == 2 && s_ticket % static_cast<uint32_t>(a.splits) != 0) {
      if (threadIdx.x == 0)
        while (ld_acquire_u32(a.sync + kTcSyncSlots + tile) < s_ticket / static_cast<uint32_t>(a.splits) + 1) {
        }
      __syncthreads();
    }
    if (TRACE && threadIdx.x == 0) tr[5] = gtime();
    if (threadIdx.x == 0) {
      fence_proxy_async_global();
      for (int b = 0; b < nbox; ++b) {
        int64_t off = b ? o1.cc : o.cc;
        const int co0 = static_cast<int>(off % a.oshape[3]);
        off /= a.oshape[3];
        const int q0 = static_cast<int>(off % a.oshape[2]);
        off /= a.oshape[2];
        const int p0 = static_cast<int>(off % a.oshape[1]);
        const int n0 = static_cast<int>(off / a.oshape[1]);
        for (int c0 = 0; c0 < a.bn; c0 += 32) {
          const uint32_t src = base + (b * nch + c0 / 32) * 8192;
          if constexpr (MODE == 2) tma_reduce_add_4d(&tmc, src, co0 + c0, q0, p0, n0);
          else tma_store_4d(&tmc, src, co0 + c0, q0, p0, n0);
        }
      }
      bulk_commit();
      bulk_wait_all();
    }
  } else {
    if (row < live) {
      float* stg = reinterpret_cast<float*>(gbase) + row * red_ld;
      for (int c0 = 0; c0 < a.bn; c0 += 16) {
        float v[16];
        tmem_ld16(tmem + (static_cast<uint32_t>(warp * 32) << 16) + c0, v);
#pragma unroll
        for (int q = 0; q < 4; ++q)
          *reinterpret_cast<float4*>(stg + c0 + 4 * q) =
              make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
      }
    }
    __syncthreads();
    if (TRACE && threadIdx.x == 0) tr[4] = gtime();
    if (MODE == 2 && s_ticket % static_cast<uint32_t>(a.splits) != 0) {
      if (threadIdx.x == 0)
        while (ld_acquire_u32(a.sync + kTcSyncSlots + tile) < s_ticket / static_cast<uint32_t>(a.splits) + 1) {
        }
      __syncthreads();
    }
    if (TRACE && threadIdx.x == 0) tr[5] = gtime();
    const float* sb = reinterpret_cast<const float*>(gbase);
    for (int e = threadIdx.x; e < live * c4; e += 128) {
      const int r = e / c4, cc = (e % c4) * 4;
      const float4 v = *reinterpret_cast<const float4*>(sb + r * red_ld + cc);
      if constexpr (MODE == 2) red_add_f4(out_row(r) + cc, v);
      else *reinterpret_cast<float4*>(out_row(r) + cc) = v;
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

using ConvKernel = void (*)(CUtensorMap, CUtensorMap, CUtensorMap, TcConvArgs);

template <bool TRACE, bool X3>
ConvKernel pick_conv_t(int mode, bool tma_epi) {
  if constexpr (!X3) {
    if (mode == 1) return tc_conv_kernel<1, false, TRACE, false>;
  } else {
    if (mode == 1) return nullptr;
  }
  if (mode == 2) return tma_epi ? tc_conv_kernel<2, true, TRACE, X3> : tc_conv_kernel<2, false, TRACE, X3>;
  return tma_epi ? tc_conv_kernel<0, true, TRACE, X3> : tc_conv_kernel<0, false, TRACE, X3>;
}

ConvKernel pick_conv(int mode, bool tma_epi, bool trace, bool x3) {
  if (x3) return trace ? pick_conv_t<true, true>(mode, tma_epi) : pick_conv_t<false, true>(mode, tma_epi);
  return trace ? pick_conv_t<true, false>(mode, tma_epi) : pick_conv_t<false, false>(mode, tma_epi);
}

// smem opt-in (and the non-portable cluster size of the mode-1 kernels) of
// every instantiation, once
int conv_max_dyn() {
  static int max_dyn = [] {
    int m = 1 << 30;
    for (int mode : {0, 1, 2})
      for (bool epi : {false, true})
        for (bool t : {false, true})
          for (bool x3 : {false, true}) {
            if (mode == 1 && (epi || x3)) continue;
            const void* fn = reinterpret_cast<const void*>(pick_conv(mode, epi, t, x3));
            m = std::min(m, opt_in_dynamic_smem(fn));
            if (mode == 1 && cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess) {
              cudaGetLastError();
              m = -1;
            }
          }
    return m;
  }();
  return max_dyn;
}

}  // namespace

void preload_tc_conv() { conv_max_dyn(); }

bool launch_tc_conv(const void* tmap_x, const void* tmap_w, float* c, const TcConvCfg& g, bool pdl,
                    cudaStream_t st, unsigned long long* trace, uint32_t* sync, const void* tmap_c,
                    const int64_t* oshape, int x_images) {
  const int max_dyn = conv_max_dyn();
  if (max_dyn <= 0 || g.smem_bytes > max_dyn) return false;
  if (g.splits > kMaxClusterSplits || g.grid_m > 65535 || g.grid_n > 65535) return false;
  if (g.splits * g.kt > kConvMaxK) return false;
  TcConvArgs a;
  a.c = c;
  a.trace = trace;
  a.m_grid = g.m_grid;
  a.n_grid = g.n_grid;
  a.x_n0 = g.x_n0; a.x_h0 = g.x_h0; a.x_w0 = g.x_w0; a.x_c0 = g.x_c0;
  a.c0 = g.c0; a.cc_h1 = g.cc_h1; a.cc_w1 = g.cc_w1;
  for (int64_t sp = 0; sp < g.splits; ++sp)
    for (int64_t kt = 0; kt < g.kt; ++kt) {
      Coord t{0, 0, 0, 0, 0, 0, 0};
      host_add_parts(g.k_split, sp, t);
      host_add_parts(g.k_tile, kt, t);
      KCoord& k = a.kc[sp * g.kt + kt];
      k.c = static_cast<int32_t>(t.c);
      k.w = static_cast<int32_t>(t.w);
      k.h = static_cast<int32_t>(t.h);
      k.n = static_cast<int32_t>(t.n);
      k.kf = static_cast<int32_t>(t.kf);
      k.pad = 0;
    }
  a.bn = static_cast<int>(g.bn);
  a.splits = static_cast<int>(g.splits);
  a.kt = static_cast<int>(g.kt);
  a.stages = static_cast<int>(g.stages);
  // split-K: L2 reduction with arrival tickets (mode 2) when the runner gave
  // ticket slots; the cluster DSMEM reduction (mode 1) otherwise
  a.mode = g.splits == 1 ? 0 : (sync && g.grid_m * g.grid_n <= kTcSyncSlots ? 2 : 1);
  if (g.x3 && (a.mode == 1 || x_images <= 0)) return false;  // 3xTF32: L2 split-K only
  a.lo_n = g.x3 ? x_images : 0;
  a.sync = sync;
  // TMA epilogue: the 64 box rows are the 8 x 8 pixels of an NHWC output
  // ([n][p][q][k], row r -> (p0 + r/8, q0 + r%8)) and BN is whole 32-ch chunks
  a.tma_epi = 0;
  if (tmap_c && oshape && a.mode != 1 && g.bn % 32 == 0 && g.cc_w1 == oshape[3] &&
      g.cc_h1 == oshape[2] * oshape[3]) {
    a.tma_epi = 1;
    for (int d = 0; d < 4; ++d) a.oshape[d] = oshape[d];
  }
  const uint32_t fmt = g.x3 ? 2u : 1u;  // tf32 : bf16 operands
  a.idesc = (1u << 4) | (fmt << 7) | (fmt << 10) | (static_cast<uint32_t>(g.bn >> 3) << 17) |
            (static_cast<uint32_t>(128 >> 4) << 24);
  uint32_t cols = 32;
  while (cols < static_cast<uint32_t>(g.bn)) cols <<= 1;
  a.tmem_cols = cols;
  // box pairs: every UMMA row live, half the CTAs; needs the doubled staged
  // tile to fit beside the ring the planner sized
  a.grid_m = static_cast<int>(g.grid_m);
  {
    const int64_t ring = g.stages * (kStageA + g.bn * 64 * 2);
    const int64_t tile2 = 2LL * kRows * (g.bn + 4) * 4;
    const int64_t need = 1024 + std::max(ring, tile2) + 16 * g.stages + 64;
    // measured (profiles/r02_conv_pairs.txt): pairing pays for the narrow
    // BN 16 tiles (15.6 vs 20.6 us, 18.6 vs 24.7 us) and for grids of more
    // than two CTAs per SM; for BN >= 32 at <= 2 CTAs per SM the extra CTAs
    // hide more latency than the dead half-rows cost
    const int64_t ctas = g.grid_m * g.grid_n * g.splits;
    a.pair = !g.x3 && a.mode != 1 && g.grid_m > 1 && need <= g.smem_bytes && (g.bn <= 16 || ctas > 2 * 148) ? 1 : 0;
  }
  const int64_t grid_y = a.pair ? (g.grid_m + 1) / 2 : g.grid_m;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(g.grid_n), static_cast<unsigned>(grid_y), static_cast<unsigned>(g.splits));
  cfg.blockDim = dim3(128, 1, 1);
  cfg.dynamicSmemBytes = static_cast<size_t>(g.smem_bytes);
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
  attr[1].id = cudaLaunchAttributeClusterDimension;  // mode 1 only: a 1x1x1 cluster launch costs time
  attr[1].val.clusterDim.x = 1;
  attr[1].val.clusterDim.y = 1;
  attr[1].val.clusterDim.z = static_cast<unsigned>(g.splits);
  cfg.attrs = attr;
  cfg.numAttrs = a.mode == 1 ? 2 : 1;
  const CUtensorMap tx = *static_cast<const CUtensorMap*>(tmap_x);
  const CUtensorMap tw = *static_cast<const CUtensorMap*>(tmap_w);
  const CUtensorMap tcm = a.tma_epi ? *static_cast<const CUtensorMap*>(tmap_c) : tw;
  const ConvKernel kern = pick_conv(a.mode, a.tma_epi != 0, trace != nullptr, g.x3);
  if (!kern) return false;
  if (cudaLaunchKernelEx(&cfg, kern, tx, tw, tcm, a) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return cudaGetLastError() == cudaSuccess;
}

}  // namespace lsb
