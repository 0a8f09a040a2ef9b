// TCGEN05 family: one 128 x BN UMMA tile per CTA, bf16 operands staged by TMA
// into 128-byte-swizzled shared memory, fp32 accumulator in TMEM.
//
// Warp roles (128 threads):
//   warp 0  : TMEM allocation; lane 0 is the TMA producer
//   warp 1  : lane 0 initialises the mbarriers and issues tcgen05.mma
//   warps 0-3: epilogue -- tcgen05.ld of their 32 TMEM lanes (= 32 output
//             rows) into a padded shared-memory tile over the finished ring.
// Launched with programmatic dependent launch: setup (TMEM allocation,
// barrier init, descriptor prefetch) overlaps the previous grid's tail and
// griddepcontrol.wait guards every global access.
// The k loop is an S-stage smem ring: full[s] (TMA tx-count) and empty[s]
// (tcgen05.commit) mbarriers.
//
// Split-K (plan.hpp tc_geom): the CTAs of one tile form clusters of `cl`
// (cluster dims 1 x 1 x cl).  After the MMAs each CTA stages its partial tile
// in its own shared memory and pushes row slice o to cluster peer o with one
// bulk DSMEM copy (cp.async.bulk shared::cluster, completing tx bytes on the
// peer's receive mbarrier) -- a reduce-scatter with no cluster-wide barrier
// on the critical path; each CTA then sums its slice and writes it once.
// With more than one cluster per tile (splits > 16) the cluster partials of a
// slice meet in global memory: an arrival ticket (per-candidate counter,
// never reset within a candidate, so launch L owns tickets [L*parts,
// (L+1)*parts)) lets the first arriver store and the others red.add after
// its release flag -- no memset node between launches.
// Instantiated at runtime for any BN in [16, 256] step 16, split-K ways,
// k-tiles and stage count (see plan.cpp).
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include "kernels.cuh"
#include "tc_common.cuh"

namespace lsb {

namespace {

using namespace tc;

struct TcArgs {
  float* c;
  int64_t sc_b, sc_m;
  int bn, splits, kt, stages;
  int mode, cl, parts, rows_per, ld;
  int mc;                     // cluster of N-tiles sharing A by TMA multicast (cluster dims mc x 1 x cl)
  int debug;                  // experiment knob LSB_TC_DEBUG: 1 skip loads+MMA, 2 skip the epilogue,
                              // 4 skip the C stores, 8 skip the cluster exchange
  int reg_epi;                // mode 0, LSB_TC_REGEPI=1: registers -> global directly
  int tma_epi;                // modes 0/2, BN % 32 == 0: 128B-swizzled 32-column chunks, TMA store / add-reduce
  int full_wait;              // wait for TMA store / reduce completion before exit (LSB_TC_STOREWAIT=0: smem reads only)
  int early_poll;             // mode 2: observe the zeroing flag during the main loop (LSB_TC_EARLYPOLL)
  int direct;                 // push rows from registers (st.shared::cluster) instead of staged bulk copies
  uint32_t ring_or_tile;      // bytes from the aligned base to the receive buffer
  uint32_t* sync;             // mode 2: [kTcSyncSlots] tickets, then [kTcSyncSlots] ready flags
  unsigned long long* trace;  // optional per-CTA globaltimer stamps (8 per CTA)
  uint32_t idesc;
  uint32_t tmem_cols;
};

constexpr int kTile = 128 * 64 * 2;  // A stage bytes

__global__ void __launch_bounds__(128, 1)
tc_gemm_kernel(const __grid_constant__ CUtensorMap tma, const __grid_constant__ CUtensorMap tmb,
               const __grid_constant__ CUtensorMap tmc, TcArgs a) {
  extern __shared__ uint8_t smem_raw[];
  __shared__ uint32_t s_ticket;
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* gbase = smem_raw + (base - raw);
  const int b_bytes = a.bn * 64 * 2;
  const uint32_t a0 = base;                     // A stages
  const uint32_t b0 = base + a.stages * kTile;  // B stages
  const uint32_t recv = base + a.ring_or_tile;  // peers' slices of my rows: [cl][rows_per][ld] fp32
  const uint32_t recv_bytes = a.cl > 1 ? static_cast<uint32_t>(a.cl * a.rows_per * a.ld * 4) : 0u;
  const uint32_t bars = (recv + recv_bytes + 15u) & ~15u;
  const uint32_t full = bars, empty = bars + 8 * a.stages, done = bars + 16 * a.stages;
  const uint32_t recv_bar = done + 8;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(gbase + (bars - base) + 16 * a.stages + 16);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_blk = blockIdx.x, m_blk = blockIdx.y;
  const size_t cta = (static_cast<size_t>(blockIdx.z) * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
  unsigned long long* tr = a.trace ? a.trace + 8 * cta : nullptr;
  if (tr && threadIdx.x == 0) tr[0] = gtime();
  const int batch = blockIdx.z / a.splits, split = blockIdx.z % a.splits;
  const int me = split % a.cl;  // == %cluster_ctarank (cluster dims 1 x 1 x cl)
  const int r_lo = me * a.rows_per;
  const int nrows = max(0, min(128, r_lo + a.rows_per) - r_lo);

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(a.tmem_cols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (threadIdx.x == 32) {
    for (int s = 0; s < a.stages; ++s) {
      mbar_init(full + 8 * s, 1);
      mbar_init(empty + 8 * s, a.mc);  // every CTA of the multicast group frees the slot
    }
    mbar_init(done, 1);
    mbar_init(recv_bar, 1);
    // every peer pushes its copy of my row slice: arm the tx count up front
    if (a.cl > 1 && !a.direct) mbar_expect_tx(recv_bar, static_cast<uint32_t>((a.cl - 1) * nrows * a.ld * 4));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tma)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmb)) : "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // my barriers are initialised: peers may push / multicast into me after
  // their matching cluster wait
  if (a.cl > 1 || a.mc > 1) cluster_arrive();
  if (tr && threadIdx.x == 0) tr[1] = gtime();

  const uint32_t stage_bytes = kTile + b_bytes;
  // programmatic dependent launch: the next grid may start its prologue now;
  // this grid waits for its predecessor before its first global access
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (a.mc > 1) cluster_wait();  // (latency overlapped with griddepcontrol.wait)
  const int mrank = blockIdx.x % a.mc;
  const int a_rows = 128 / a.mc;
  const uint16_t mc_mask = static_cast<uint16_t>((1u << a.mc) - 1u);

  const int tile = (batch * gridDim.y + m_blk) * gridDim.x + n_blk;
  float* ctile = a.c + batch * a.sc_b + static_cast<int64_t>(m_blk) * 128 * a.sc_m + static_cast<int64_t>(n_blk) * a.bn;
  const int c4 = a.bn / 4;
  if (a.mode == 2 && warp >= 2) {
    // ---- mode 2: every CTA takes its arrival ticket now (off the critical
    // path); the first CTA of the tile to start zeroes it while its operands
    // stream in, the others observe the zeroing before their epilogue ----
    const int t2 = threadIdx.x - 64;
    if (t2 == 0) s_ticket = atomicAdd(a.sync + tile, 1u);
    asm volatile("bar.sync 1, 64;" ::: "memory");
    const uint32_t t = s_ticket;
    const uint32_t L = t / static_cast<uint32_t>(a.parts);
    if (t % static_cast<uint32_t>(a.parts) == 0) {
      const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int e = t2; e < 128 * c4; e += 64) {
        const int r = e / c4, cc = (e % c4) * 4;
        *reinterpret_cast<float4*>(ctile + static_cast<int64_t>(r) * a.sc_m + cc) = z;
      }
      asm volatile("bar.sync 1, 64;" ::: "memory");
      if (t2 == 0) st_release_u32(a.sync + kTcSyncSlots + tile, L + 1);  // cumulative over the barrier
    } else if (t2 == 0 && a.early_poll) {
      // first poll once the last k-tile has landed; back off between polls
      const int last = a.kt - 1;
      if (!(a.debug & 1)) mbar_wait(full + 8 * (last % a.stages), (last / a.stages) & 1);
      while (ld_acquire_u32(a.sync + kTcSyncSlots + tile) < L + 1) __nanosleep(64);
    }
  }

  if (a.debug & 1) {
    if (threadIdx.x == 32) umma_commit(done);
  } else if (warp == 0 && lane == 0) {
    // ---- TMA producer ----
    for (int kt = 0; kt < a.kt; ++kt) {
      const int s = kt % a.stages;
      const uint32_t ph = (kt / a.stages) & 1;
      const int kc = (split * a.kt + kt) * 64;
      if (kt >= a.stages) mbar_wait(empty + 8 * s, ph ^ 1);
      mbar_expect_tx(full + 8 * s, stage_bytes);
      if (a.mc > 1)  // my 128/mc-row slice of the A k-tile, into every CTA of the group
        tma_load_3d_mc(a0 + s * kTile + mrank * a_rows * 128, &tma, full + 8 * s, kc, m_blk * 128 + mrank * a_rows,
                       batch, mc_mask);
      else
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
      if (kt + a.stages < a.kt) {  // the slot is refilled: free it in every CTA that writes it
        if (a.mc > 1) umma_commit_mc(empty + 8 * s, mc_mask);
        else umma_commit(empty + 8 * s);
      }
    }
    umma_commit(done);
  }

  // ---- epilogue ----
  mbar_wait(done, 0);
  __syncwarp();
  tc_fence_after();
  if (tr && threadIdx.x == 0) tr[3] = gtime();
  if (a.debug & 2) {
    if (a.cl > 1) cluster_wait();
    if (a.mc > 1) {
      cluster_arrive();
      cluster_wait();
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0)
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(a.tmem_cols) : "memory");
    return;
  }
  const int row = warp * 32 + lane;  // TMEM lane == output row of this thread
  const uint32_t trow = tmem + (static_cast<uint32_t>(warp * 32) << 16);
  if (a.direct) {
    // tile + receive buffer exceed smem: each row goes from registers to the
    // peer that owns it (slot `me` of the owner's receive buffer)
    cluster_wait();
    const int owner = row / a.rows_per, lr = row - owner * a.rows_per;
    const uint32_t dst = map_peer(recv + static_cast<uint32_t>((me * a.rows_per + lr) * a.ld * 4), owner);
    for (int c0 = 0; c0 < a.bn; c0 += 16) {
      uint32_t v[16];
      tmem_ld16_nowait(trow + c0, v);
      tmem_wait();
#pragma unroll
      for (int q = 0; q < 4; ++q)
        st_cluster_f4(dst + static_cast<uint32_t>((c0 + 4 * q) * 4), __uint_as_float(v[4 * q]),
                      __uint_as_float(v[4 * q + 1]), __uint_as_float(v[4 * q + 2]), __uint_as_float(v[4 * q + 3]));
    }
    cluster_arrive();
    cluster_wait();  // every pushed row has landed
  } else if (a.reg_epi) {
    // mode 0 experiment (LSB_TC_REGEPI=1): rows straight from TMEM registers
    // to global (no smem staging, no bulk-store wait before exit)
    float* crow = a.c + batch * a.sc_b + (static_cast<int64_t>(m_blk) * 128 + row) * a.sc_m +
                  static_cast<int64_t>(n_blk) * a.bn;
    for (int c0 = 0; c0 < a.bn; c0 += 16) {
      uint32_t v[16];
      tmem_ld16_nowait(trow + c0, v);
      tmem_wait();
#pragma unroll
      for (int q = 0; q < 4; ++q)
        *reinterpret_cast<float4*>(crow + c0 + 4 * q) =
            make_float4(__uint_as_float(v[4 * q]), __uint_as_float(v[4 * q + 1]), __uint_as_float(v[4 * q + 2]),
                        __uint_as_float(v[4 * q + 3]));
    }
  } else if (a.tma_epi) {
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
    __syncthreads();
  } else {
    // TMEM -> padded smem tile over the finished ring
    float* stg = reinterpret_cast<float*>(gbase) + row * a.ld;
    int c0 = 0;
    for (; c0 + 32 <= a.bn; c0 += 32) {
      uint32_t v[32];
      tmem_ld16_nowait(trow + c0, v);
      tmem_ld16_nowait(trow + c0 + 16, v + 16);
      tmem_wait();
#pragma unroll
      for (int q = 0; q < 8; ++q)
        *reinterpret_cast<float4*>(stg + c0 + 4 * q) =
            make_float4(__uint_as_float(v[4 * q]), __uint_as_float(v[4 * q + 1]), __uint_as_float(v[4 * q + 2]),
                        __uint_as_float(v[4 * q + 3]));
    }
    if (c0 < a.bn) {
      uint32_t v[16];
      tmem_ld16_nowait(trow + c0, v);
      tmem_wait();
#pragma unroll
      for (int q = 0; q < 4; ++q)
        *reinterpret_cast<float4*>(stg + c0 + 4 * q) =
            make_float4(__uint_as_float(v[4 * q]), __uint_as_float(v[4 * q + 1]), __uint_as_float(v[4 * q + 2]),
                        __uint_as_float(v[4 * q + 3]));
    }
    if (a.cl > 1) fence_proxy_async_smem();  // staged rows are read by the bulk-copy engine
    __syncthreads();
  }
  if (tr && threadIdx.x == 0) tr[4] = gtime();

  const float* stile = reinterpret_cast<const float*>(gbase);
  if (a.reg_epi) {
    // stored above
  } else if (a.mode != 1) {
    if (a.mode == 2 && !a.early_poll && s_ticket % static_cast<uint32_t>(a.parts) != 0) {
      if (threadIdx.x == 0)
        while (ld_acquire_u32(a.sync + kTcSyncSlots + tile) < s_ticket / static_cast<uint32_t>(a.parts) + 1) {
        }
      __syncthreads();
    }
    if (tr && threadIdx.x == 0) tr[5] = gtime();
    if (a.tma_epi) {
      if (threadIdx.x == 0) {
        fence_proxy_async_global();  // the (acquired) zeroing precedes the async-proxy reduction
        for (int c0 = 0; c0 < a.bn; c0 += 32) {
          const uint32_t src = base + (c0 / 32) * 16384;
          if (a.mode == 0) tma_store_3d(&tmc, src, n_blk * a.bn + c0, m_blk * 128, batch);
          else tma_reduce_add_3d(&tmc, src, n_blk * a.bn + c0, m_blk * 128, batch);
        }
        bulk_commit();
        if (a.full_wait) bulk_wait_all();
        else bulk_wait_read();
      }
    } else
    for (int e = threadIdx.x; e < 128 * c4; e += 128) {
      const int r = e / c4, cc = (e % c4) * 4;
      const float4 acc = *reinterpret_cast<const float4*>(stile + r * a.ld + cc);
      float* dst = ctile + static_cast<int64_t>(r) * a.sc_m + cc;
      if ((a.debug & 4) && acc.x != -12345.f) continue;
      if (a.mode == 0) *reinterpret_cast<float4*>(dst) = acc;
      else red_add_f4(dst, acc);
    }
  } else {
    const bool xchg = a.cl > 1 && !a.direct && !(a.debug & 8);
    if (xchg) {
      // ---- reduce-scatter inside the cluster: push slice o to peer o ----
      cluster_wait();  // every peer's receive barrier is initialised
      if (threadIdx.x == 0) {
        for (int o = 0; o < a.cl; ++o) {
          if (o == me) continue;
          const int lo = o * a.rows_per, nr = min(128, lo + a.rows_per) - lo;
          if (nr <= 0) continue;
          const uint32_t bytes = static_cast<uint32_t>(nr * a.ld * 4);
          const uint32_t src = base + static_cast<uint32_t>(lo * a.ld * 4);
          const uint32_t dst = map_peer(recv + static_cast<uint32_t>(me * a.rows_per * a.ld * 4), o);
          bulk_push_peer(dst, src, bytes, map_peer(recv_bar, o));
        }
      }
      mbar_wait(recv_bar, 0);
      // all copies into me have landed: peers may exit once everyone got theirs
      cluster_arrive();
    }
    if (tr && threadIdx.x == 0) tr[5] = gtime();
    const float* rb = reinterpret_cast<const float*>(gbase + (recv - base));
    for (int e = threadIdx.x; e < nrows * c4; e += 128) {
      const int lr = e / c4, cc = (e % c4) * 4;
      float4 acc = a.direct ? *reinterpret_cast<const float4*>(rb + (me * a.rows_per + lr) * a.ld + cc)
                            : *reinterpret_cast<const float4*>(stile + (r_lo + lr) * a.ld + cc);
      for (int q = 0; q < a.cl; ++q) {
        if (q == me || (a.debug & 8)) continue;
        const float4 v = *reinterpret_cast<const float4*>(rb + (q * a.rows_per + lr) * a.ld + cc);
        acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
      }
      float* dst = ctile + static_cast<int64_t>(r_lo + lr) * a.sc_m + cc;
      if ((a.debug & 4) && acc.x != -12345.f) continue;
      *reinterpret_cast<float4*>(dst) = acc;
    }
    if (a.cl > 1 && !a.direct) cluster_wait();  // my pushes have been received: my smem may go away
  }
  if (tr && threadIdx.x == 0) {
    tr[6] = gtime();
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    tr[7] = smid;
  }
  if (a.mc > 1) {  // no multicast write or remote arrival may target an exited CTA
    cluster_arrive();
    cluster_wait();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(a.tmem_cols) : "memory");
  }
}

}  // namespace

void preload_tc_gemm() { opt_in_dynamic_smem(reinterpret_cast<const void*>(tc_gemm_kernel)); }

bool launch_tc_gemm(const TcLaunch& L, cudaStream_t st) {
  static int max_dyn = -1;
  if (max_dyn < 0) max_dyn = opt_in_dynamic_smem(reinterpret_cast<const void*>(tc_gemm_kernel));
  if (max_dyn <= 0 || L.smem_bytes > max_dyn) return false;
  const TcGeom g =
      tc_geom(L.bn, L.splits, L.stages, static_cast<int64_t>(L.batch) * L.grid_m * L.grid_n, L.grid_n);
  if (g.mode == 2 && !L.sync) return false;
  TcArgs a;
  a.c = L.c;
  a.sc_b = L.sc_b;
  a.sc_m = L.sc_m;
  a.bn = L.bn;
  a.splits = L.splits;
  a.kt = L.kt;
  a.stages = L.stages;
  a.mode = g.mode;
  a.cl = g.cl;
  a.mc = g.mc;
  a.parts = g.parts;
  a.rows_per = g.rows_per;
  a.ld = g.ld;
  static const int debug = getenv("LSB_TC_DEBUG") ? atoi(getenv("LSB_TC_DEBUG")) : 0;
  a.debug = debug;

  a.direct = L.direct ? 1 : 0;
  static const int early_poll = getenv("LSB_TC_EARLYPOLL") ? atoi(getenv("LSB_TC_EARLYPOLL")) : 0;
  a.early_poll = early_poll;
  static const int full_wait = getenv("LSB_TC_STOREWAIT") ? atoi(getenv("LSB_TC_STOREWAIT")) : 1;
  a.full_wait = full_wait;
  static const bool no_tma_epi = getenv("LSB_TC_NOTMAEPI") && atoi(getenv("LSB_TC_NOTMAEPI")) != 0;
  a.tma_epi = L.tmap_c && !no_tma_epi && (g.mode == 0 || g.mode == 2) && L.bn % 32 == 0 ? 1 : 0;
  static const bool reg_epi = getenv("LSB_TC_REGEPI") && atoi(getenv("LSB_TC_REGEPI")) != 0;
  a.reg_epi = reg_epi && g.mode == 0 && !L.trace ? 1 : 0;
  a.ring_or_tile = static_cast<uint32_t>(((L.direct ? g.ring : std::max(g.ring, g.tile)) + 15) & ~15LL);
  a.sync = L.sync;
  a.trace = L.trace;
  // kind::f16 instruction descriptor: D f32, A/B bf16, both K-major, N>>3, M>>4
  a.idesc = (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(L.bn >> 3) << 17) |
            (static_cast<uint32_t>(128 >> 4) << 24);
  uint32_t cols = 32;
  while (cols < static_cast<uint32_t>(L.bn)) cols <<= 1;
  a.tmem_cols = cols;
  static bool nonportable = false;
  if (a.cl * a.mc > 8 && !nonportable) {
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
  attr[0].val.clusterDim.x = static_cast<unsigned>(a.mc);
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = static_cast<unsigned>(a.cl);
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  static const bool nopdl = getenv("LSB_TC_NOPDL") && atoi(getenv("LSB_TC_NOPDL")) != 0;
  attr[1].val.programmaticStreamSerializationAllowed = L.pdl && !nopdl ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  const CUtensorMap ta = *static_cast<const CUtensorMap*>(L.tmap_a);
  const CUtensorMap tb = *static_cast<const CUtensorMap*>(L.tmap_b);
  const CUtensorMap tc = L.tmap_c ? *static_cast<const CUtensorMap*>(L.tmap_c) : tb;
  if (cudaLaunchKernelEx(&cfg, tc_gemm_kernel, ta, tb, tc, a) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return cudaGetLastError() == cudaSuccess;
}

}  // namespace lsb
