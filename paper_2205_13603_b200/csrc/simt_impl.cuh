// SIMT family (kernels.cu's launch_simt picks the instantiation): CTA tiles
// staged through shared memory, per-thread RM x RN register tiles, fp32
// accumulation; cp.async double-buffered k-tiles for fp32 operands.
//
// CHK selects the checked-launch variant with deadline checks inside the
// tile staging loop (a few-thread CTA staging a long tile); timed repeats use
// the CHK=false kernel without them (that code cost the best gmm512 schedule
// 15 % when compiled into the same kernel).  The cheaper checks (top of a
// k-tile, between 64-step k chunks, after the tile loop) and the persistent
// tile loop are runtime-gated on the deadline pointer in both variants.
// Instantiated in simt_{f32,bf16}_{fast,chk}.cu (compiled in parallel).
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "kernels.cuh"

namespace lsb {
namespace simt {

__device__ __forceinline__ float ldf(const float* p, int64_t i) { return __ldg(p + i); }
__device__ __forceinline__ float ldf(const __nv_bfloat16* p, int64_t i) { return __bfloat162float(p[i]); }

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

struct SArgs {
  Strides s;
  int64_t tb, tm, tn, rb, bk, kt;
  int x_kfast, y_kfast;
  int va, vb;                 // global vector width (1 or 16 bytes' worth) per operand
  int lda, ldb;               // padded smem row lengths
  int a_vec_smem, b_vec_smem; // 128-bit smem reads possible
  int c_vec;                  // 128-bit output stores possible
  int db;                     // fp32 only: cp.async double-buffered k-tiles (two smem tile sets)
  int persist;                // checked launches: one wave of CTAs loops over the tiles, so a
                              // timed-out candidate stops within one k-tile instead of draining
                              // every remaining wave of its grid
  int64_t ntn, ntm, ntb;      // tile counts (grid x, y, z of the plain launch)
  const unsigned long long* deadline;
  int* timed_out;
};

// ---- SIMT family -----------------------------------------------------------
// CTA (gn, gm, gb) owns a BM x BN output tile of tb*rb batches; thread
// (tb_i, tm_i, tn_i) owns an RM x RN register tile (rows tm_i*RM.., cols
// tn_i*RN..) of rb batches; k runs in kt shared-memory tiles of bk.
// Tiles are staged k-major in shared memory (S[tb][kk][row], rows padded when
// that breaks bank conflicts); global loads walk the operand's contiguous
// dimension with 16-byte vectors when the tile and strides allow it and use
// carried indices instead of per-element division.
template <typename T> struct VecW { static constexpr int v = 4; };
template <> struct VecW<__nv_bfloat16> { static constexpr int v = 8; };

template <typename T, int V>
__device__ __forceinline__ void ld_vec(const T* p, float* out) {
  if constexpr (V == 1) {
    out[0] = ldf(p, 0);
  } else if constexpr (sizeof(T) == 4) {
    float4 q = __ldg(reinterpret_cast<const float4*>(p));
    out[0] = q.x; out[1] = q.y; out[2] = q.z; out[3] = q.w;
  } else {
    uint4 q = __ldg(reinterpret_cast<const uint4*>(p));
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&q);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      float2 f = __bfloat1622float2(h[i]);
      out[2 * i] = f.x; out[2 * i + 1] = f.y;
    }
  }
}

// Stage one operand tile S[t][kk][r] (t < nt, kk < bk, r < nr) from global
// g[b*s_b + (r0+r)*s_r + (k0+kk)*s_k].  kfast: k is the vector/contiguous
// dimension, else r is.
template <typename T, int V>
__device__ __forceinline__ void stage_tile(float* S, int lds, const T* __restrict__ g, int64_t s_b, int64_t s_r,
                                           int64_t s_k, int64_t b0, int64_t brb, int64_t rbi, int64_t r0, int64_t k0,
                                           int nt, int nr, int bk, bool kfast, int tid, int nthr,
                                           unsigned long long dl = 0) {
  const int nf = (kfast ? bk : nr) / V;   // vectors along the fast dim
  const int ns = kfast ? nr : bk;          // slow dim
  const int total = nt * ns * nf;
  if (tid >= total) return;
  int f = tid % nf, q = tid / nf, sl = q % ns, t = q / ns;
  const int sf = nthr % nf, sq = nthr / nf, ss = sq % ns, st = sq / ns;
  int steps = 0;
  for (int e = tid; e < total; e += nthr) {
    // a CTA with few threads and a long tile checks the deadline while it
    // stages (the caller aborts after the tile's barrier)
    if (dl && (++steps & 255) == 0 && gtimer() > dl) break;
    const int64_t b = b0 + t * brb + rbi;
    float v[V];
    if (kfast) {
      const int kk = f * V, r = sl;
      ld_vec<T, V>(g + b * s_b + (r0 + r) * s_r + (k0 + kk) * s_k, v);
      float* d = S + (t * bk + kk) * lds + r;
#pragma unroll
      for (int i = 0; i < V; ++i) d[i * lds] = v[i];
    } else {
      const int r = f * V, kk = sl;
      ld_vec<T, V>(g + b * s_b + (r0 + r) * s_r + (k0 + kk) * s_k, v);
      float* d = S + (t * bk + kk) * lds + r;
#pragma unroll
      for (int i = 0; i < V; ++i) d[i] = v[i];
    }
    f += sf;
    int c = 0;
    if (f >= nf) { f -= nf; c = 1; }
    sl += ss + c;
    c = 0;
    if (sl >= ns) { sl -= ns; c = 1; }
    t += st + c;
  }
}

__device__ __forceinline__ void cp_async4(float* dst, const float* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
               "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async16(float* dst, const float* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
               "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// stage_tile for fp32 operands without a register round trip: the same index
// walk, every element (or 16-byte run along the tile's row when rows are
// 16-byte aligned in smem) is a cp.async, so the next k-tile streams in while
// the current one is computed
template <int V>
__device__ __forceinline__ void stage_tile_async(float* S, int lds, const float* __restrict__ g, int64_t s_b,
                                                 int64_t s_r, int64_t s_k, int64_t b0, int64_t brb, int64_t rbi,
                                                 int64_t r0, int64_t k0, int nt, int nr, int bk, bool kfast, int tid,
                                                 int nthr) {
  const int nf = (kfast ? bk : nr) / V;
  const int ns = kfast ? nr : bk;
  const int total = nt * ns * nf;
  if (tid >= total) return;
  int f = tid % nf, q = tid / nf, sl = q % ns, t = q / ns;
  const int sf = nthr % nf, sq = nthr / nf, ss = sq % ns, st = sq / ns;
  const bool row16 = V == 4 && (lds % 4) == 0;
  for (int e = tid; e < total; e += nthr) {
    const int64_t b = b0 + t * brb + rbi;
    if (kfast) {
      const int kk = f * V, r = sl;
      const float* src = g + b * s_b + (r0 + r) * s_r + (k0 + kk) * s_k;
      float* d = S + (t * bk + kk) * lds + r;
#pragma unroll
      for (int i = 0; i < V; ++i) cp_async4(d + i * lds, src + i * s_k);
    } else {
      const int r = f * V, kk = sl;
      const float* src = g + b * s_b + (r0 + r) * s_r + (k0 + kk) * s_k;
      float* d = S + (t * bk + kk) * lds + r;
      if (row16) {
        cp_async16(d, src);
      } else {
#pragma unroll
        for (int i = 0; i < V; ++i) cp_async4(d + i, src + i * s_r);
      }
    }
    f += sf;
    int c = 0;
    if (f >= nf) { f -= nf; c = 1; }
    sl += ss + c;
    c = 0;
    if (sl >= ns) { sl -= ns; c = 1; }
    t += st + c;
  }
}

template <typename T, int RM, int RN, bool CHK>
__global__ void __launch_bounds__(1024) simt_gemm(const T* __restrict__ x, const T* __restrict__ y,
                                                  float* __restrict__ c, SArgs a) {
  extern __shared__ float sm[];
  __shared__ int abort_flag;
  constexpr int VW = VecW<T>::v;
  const int tid = threadIdx.x;
  const int nthr = (int)(a.tb * a.tm * a.tn);
  const int tn_i = tid % (int)a.tn;
  const int tm_i = (tid / (int)a.tn) % (int)a.tm;
  const int tb_i = tid / (int)(a.tn * a.tm);
  const int bm = (int)a.tm * RM, bn = (int)a.tn * RN, bk = (int)a.bk;
  const int lda = a.lda, ldb = a.ldb;
  const int64_t a_words = (a.tb * bk * lda + 3) & ~(int64_t)3;  // 16-byte aligned B tile
  const int64_t set_words = (a_words + a.tb * bk * ldb + 3) & ~(int64_t)3;
  float* As = sm;
  float* Bs = sm + a_words;
  const Strides& s = a.s;
  const bool persist = a.persist;
  const int64_t ntiles = persist ? a.ntn * a.ntm * a.ntb : 1;
  for (int64_t tile = persist ? blockIdx.x : 0; tile < ntiles; tile += persist ? gridDim.x : 1) {
  int64_t bx = blockIdx.x, by = blockIdx.y, bz = blockIdx.z;
  if (persist) {
    bx = tile % a.ntn;
    by = (tile / a.ntn) % a.ntm;
    bz = tile / (a.ntn * a.ntm);
    __syncthreads();  // the previous tile's last smem reads are done
  }
  const int64_t m0 = by * bm, n0 = bx * bn;
  const int64_t b0 = bz * a.tb * a.rb;

  for (int64_t rbi = 0; rbi < a.rb; ++rbi) {
    float acc[RM][RN];
#pragma unroll
    for (int i = 0; i < RM; ++i)
#pragma unroll
      for (int j = 0; j < RN; ++j) acc[i][j] = 0.f;

    bool async_tiles = false;
    if constexpr (sizeof(T) == 4) async_tiles = a.db != 0;
    auto issue_async = [&](int64_t kti, int buf) {
      if constexpr (sizeof(T) == 4) {
        float* A2 = sm + buf * set_words;
        float* B2 = A2 + a_words;
        const int64_t k0 = kti * bk;
        if (a.va > 1)
          stage_tile_async<VW>(A2, lda, reinterpret_cast<const float*>(x), s.sx[0], s.sx[1], s.sx[3], b0, a.rb, rbi,
                               m0, k0, (int)a.tb, bm, bk, a.x_kfast, tid, nthr);
        else
          stage_tile_async<1>(A2, lda, reinterpret_cast<const float*>(x), s.sx[0], s.sx[1], s.sx[3], b0, a.rb, rbi,
                              m0, k0, (int)a.tb, bm, bk, a.x_kfast, tid, nthr);
        if (a.vb > 1)
          stage_tile_async<VW>(B2, ldb, reinterpret_cast<const float*>(y), s.sy[0], s.sy[2], s.sy[3], b0, a.rb, rbi,
                               n0, k0, (int)a.tb, bn, bk, a.y_kfast, tid, nthr);
        else
          stage_tile_async<1>(B2, ldb, reinterpret_cast<const float*>(y), s.sy[0], s.sy[2], s.sy[3], b0, a.rb, rbi,
                              n0, k0, (int)a.tb, bn, bk, a.y_kfast, tid, nthr);
      }
      cp_async_commit();
    };
    if (async_tiles) issue_async(0, 0);
    const unsigned long long dstage = CHK && a.deadline ? *a.deadline : 0ull;

    for (int64_t kti = 0; kti < a.kt; ++kti) {
      if (a.deadline) {
        if (tid == 0) abort_flag = gtimer() > *a.deadline;
        __syncthreads();
        if (abort_flag) {
          if (tid == 0) atomicExch(a.timed_out, 1);
          if (async_tiles) cp_async_wait<0>();
          return;
        }
      }
      const int64_t k0 = kti * bk;
      if (async_tiles) {
        // tile kti was issued one iteration ago; issue kti+1 into the other set
        if (kti + 1 < a.kt) {
          issue_async(kti + 1, (int)((kti + 1) & 1));
          cp_async_wait<1>();
        } else {
          cp_async_wait<0>();
        }
        As = sm + (kti & 1) * set_words;
        Bs = As + a_words;
      } else {
        if (a.va > 1)
          stage_tile<T, VW>(As, lda, x, s.sx[0], s.sx[1], s.sx[3], b0, a.rb, rbi, m0, k0, (int)a.tb, bm, bk,
                            a.x_kfast, tid, nthr, dstage);
        else
          stage_tile<T, 1>(As, lda, x, s.sx[0], s.sx[1], s.sx[3], b0, a.rb, rbi, m0, k0, (int)a.tb, bm, bk,
                           a.x_kfast, tid, nthr, dstage);
        if (a.vb > 1)
          stage_tile<T, VW>(Bs, ldb, y, s.sy[0], s.sy[2], s.sy[3], b0, a.rb, rbi, n0, k0, (int)a.tb, bn, bk,
                            a.y_kfast, tid, nthr, dstage);
        else
          stage_tile<T, 1>(Bs, ldb, y, s.sy[0], s.sy[2], s.sy[3], b0, a.rb, rbi, n0, k0, (int)a.tb, bn, bk,
                           a.y_kfast, tid, nthr, dstage);
      }
      __syncthreads();
      if (CHK && dstage && !async_tiles) {  // the staging may have stopped at the deadline
        if (tid == 0) abort_flag = gtimer() > dstage;
        __syncthreads();
        if (abort_flag) {
          if (tid == 0) atomicExch(a.timed_out, 1);
          return;
        }
      }
      const float* Ap = As + (int64_t)tb_i * bk * lda + tm_i * RM;
      const float* Bp = Bs + (int64_t)tb_i * bk * ldb + tn_i * RN;
      // checked launches look at the clock between 64-step chunks of a long
      // k-tile (the inner loop itself stays check-free)
      const unsigned long long dlv = a.deadline ? *a.deadline : 0ull;
      for (int kc = 0; kc < bk; kc += 64) {
      if (a.deadline && kc && gtimer() > dlv) break;
      const int kend = min(bk, kc + 64);
#pragma unroll 8
      for (int kk = kc; kk < kend; ++kk) {
        float av[RM], bv[RN];
        if constexpr (RM % 4 == 0) {
          if (a.a_vec_smem) {
#pragma unroll
            for (int i = 0; i < RM; i += 4) {
              float4 q = *reinterpret_cast<const float4*>(Ap + kk * lda + i);
              av[i] = q.x; av[i + 1] = q.y; av[i + 2] = q.z; av[i + 3] = q.w;
            }
          } else {
#pragma unroll
            for (int i = 0; i < RM; ++i) av[i] = Ap[kk * lda + i];
          }
        } else {
#pragma unroll
          for (int i = 0; i < RM; ++i) av[i] = Ap[kk * lda + i];
        }
        if constexpr (RN % 4 == 0) {
          if (a.b_vec_smem) {
#pragma unroll
            for (int j = 0; j < RN; j += 4) {
              float4 q = *reinterpret_cast<const float4*>(Bp + kk * ldb + j);
              bv[j] = q.x; bv[j + 1] = q.y; bv[j + 2] = q.z; bv[j + 3] = q.w;
            }
          } else {
#pragma unroll
            for (int j = 0; j < RN; ++j) bv[j] = Bp[kk * ldb + j];
          }
        } else {
#pragma unroll
          for (int j = 0; j < RN; ++j) bv[j] = Bp[kk * ldb + j];
        }
#pragma unroll
        for (int i = 0; i < RM; ++i)
#pragma unroll
          for (int j = 0; j < RN; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
      }
      }  // 64-step chunks
      __syncthreads();
    }
    if (a.deadline) {  // finished past the deadline: a timeout (no timed repeats)
      if (tid == 0) abort_flag = gtimer() > *a.deadline;
      __syncthreads();
      if (abort_flag) {
        if (tid == 0) atomicExch(a.timed_out, 1);
        return;
      }
    }
    const int64_t b = b0 + tb_i * a.rb + rbi;
    float* crow = c + b * s.sc[0] + (m0 + tm_i * RM) * s.sc[1] + (n0 + tn_i * RN) * s.sc[2];
#pragma unroll
    for (int i = 0; i < RM; ++i) {
      if constexpr (RN % 4 == 0) {
        if (a.c_vec) {
#pragma unroll
          for (int j = 0; j < RN; j += 4)
            *reinterpret_cast<float4*>(crow + i * s.sc[1] + j) = make_float4(acc[i][j], acc[i][j + 1], acc[i][j + 2], acc[i][j + 3]);
          continue;
        }
      }
#pragma unroll
      for (int j = 0; j < RN; ++j) crow[i * s.sc[1] + j * s.sc[2]] = acc[i][j];
    }
  }
  }  // tile loop
}

template <typename T, int RM, int RN, bool CHK>
cudaError_t simt_launch(const void* x, const void* y, float* c, const SArgs& a, dim3 grid, int threads, size_t smem,
                        cudaStream_t st) {
  auto fn = simt_gemm<T, RM, RN, CHK>;
  if (smem == static_cast<size_t>(-1)) {  // preload: force the (lazily loaded) function in now
    cudaFuncAttributes at;
    return cudaFuncGetAttributes(&at, fn);
  }
  static int max_dyn = -1;  // per instantiation: opt-in limit minus the kernel's static smem
  if (max_dyn < 0) {
    max_dyn = opt_in_dynamic_smem(reinterpret_cast<const void*>(fn));
    if (max_dyn <= 0) return cudaErrorInvalidValue;
  }
  if (smem > static_cast<size_t>(max_dyn)) return cudaErrorInvalidValue;
  if (CHK && a.persist) {
    static int sms = 0;
    if (!sms) {
      int dev = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    }
    // occupancy per (threads, smem) of this instantiation, cached (the query
    // costs host time on every checked launch otherwise)
    static thread_local int c_threads = -1, c_per_sm = 1;
    static thread_local size_t c_smem = 0;
    int per_sm = c_per_sm;
    if (threads != c_threads || smem != c_smem) {
      per_sm = 0;
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, threads, smem) != cudaSuccess || per_sm < 1) {
        cudaGetLastError();
        per_sm = 1;
      }
      c_threads = threads;
      c_smem = smem;
      c_per_sm = per_sm;
    }
    const int64_t tiles = static_cast<int64_t>(grid.x) * grid.y * grid.z;
    const int64_t wave = static_cast<int64_t>(sms) * per_sm;
    if (tiles > wave) {
      SArgs p = a;
      p.ntn = grid.x;
      p.ntm = grid.y;
      p.ntb = grid.z;
      fn<<<dim3(static_cast<unsigned>(wave)), threads, smem, st>>>(static_cast<const T*>(x),
                                                                   static_cast<const T*>(y), c, p);
      return cudaGetLastError();
    }
  }
  SArgs p = a;
  p.persist = 0;
  fn<<<grid, threads, smem, st>>>(static_cast<const T*>(x), static_cast<const T*>(y), c, p);
  return cudaGetLastError();
}

typedef cudaError_t (*SimtLauncher)(const void*, const void*, float*, const SArgs&, dim3, int, size_t, cudaStream_t);

// only RM x RN <= 64 is instantiated (plan.hpp kSimtTiles)
template <typename T, int RM, int RN, bool CHK>
SimtLauncher pick() {
  if constexpr (RM * RN <= 64) return simt_launch<T, RM, RN, CHK>;
  else return nullptr;
}

template <typename T, int RM, bool CHK>
void fill_row(SimtLauncher* row) {
  row[0] = pick<T, RM, 1, CHK>();
  row[1] = pick<T, RM, 2, CHK>();
  row[2] = pick<T, RM, 3, CHK>();
  row[3] = pick<T, RM, 4, CHK>();
  row[4] = pick<T, RM, 6, CHK>();
  row[5] = pick<T, RM, 8, CHK>();
  row[6] = pick<T, RM, 12, CHK>();
  row[7] = pick<T, RM, 16, CHK>();
  row[8] = pick<T, RM, 24, CHK>();
  row[9] = pick<T, RM, 32, CHK>();
  row[10] = pick<T, RM, 48, CHK>();
  row[11] = pick<T, RM, 64, CHK>();
}

template <typename T, bool CHK>
struct SimtTable {
  SimtLauncher t[12][12];
  SimtTable() {
    fill_row<T, 1, CHK>(t[0]);
    fill_row<T, 2, CHK>(t[1]);
    fill_row<T, 3, CHK>(t[2]);
    fill_row<T, 4, CHK>(t[3]);
    fill_row<T, 6, CHK>(t[4]);
    fill_row<T, 8, CHK>(t[5]);
    fill_row<T, 12, CHK>(t[6]);
    fill_row<T, 16, CHK>(t[7]);
    fill_row<T, 24, CHK>(t[8]);
    fill_row<T, 32, CHK>(t[9]);
    fill_row<T, 48, CHK>(t[10]);
    fill_row<T, 64, CHK>(t[11]);
  }
};

SimtLauncher launcher_f32_fast(int i, int j);
SimtLauncher launcher_f32_chk(int i, int j);
SimtLauncher launcher_bf16_fast(int i, int j);
SimtLauncher launcher_bf16_chk(int i, int j);

}  // namespace simt
}  // namespace lsb
