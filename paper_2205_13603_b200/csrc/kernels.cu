// Runner kernels: reference output, NAIVE / SIMT / LOOPNEST candidate
// families, K6 parity reducer and timing utilities.  The tcgen05 family lives
// in tc_gemm.cu.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>

#include "kernels.cuh"

namespace lsb {

namespace {

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

// ---- reference / naive: one thread per output element ---------------------
template <typename T, typename Acc, typename Out>
__global__ void contract_naive(const T* __restrict__ x, const T* __restrict__ y, Out* __restrict__ c, Strides s) {
  const int64_t total = s.ext[0] * s.ext[1] * s.ext[2];
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t n = e % s.ext[2], r = e / s.ext[2];
    int64_t m = r % s.ext[1], b = r / s.ext[1];
    const int64_t xo = b * s.sx[0] + m * s.sx[1], yo = b * s.sy[0] + n * s.sy[2];
    Acc acc = 0;
    for (int64_t k = 0; k < s.ext[3]; ++k)
      acc += (Acc)ldf(x, xo + k * s.sx[3]) * (Acc)ldf(y, yo + k * s.sy[3]);
    c[b * s.sc[0] + m * s.sc[1] + n * s.sc[2]] = (Out)acc;
  }
}

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

template <typename T, int RM, int RN>
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
  const int64_t ntiles = a.persist ? a.ntn * a.ntm * a.ntb : 1;
  for (int64_t tile = a.persist ? blockIdx.x : 0; tile < ntiles; tile += a.persist ? gridDim.x : 1) {
  int64_t bx = blockIdx.x, by = blockIdx.y, bz = blockIdx.z;
  if (a.persist) {
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
    const unsigned long long dstage = a.deadline ? *a.deadline : 0ull;

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
      if (dstage && !async_tiles) {  // the staging may have stopped at the deadline
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

// ---- LOOPNEST family ---------------------------------------------------------
struct NArgs {
  LoopNestCfg n;
  const unsigned long long* deadline;
  int* timed_out;
};

template <typename T>
__global__ void loopnest_contract(const T* __restrict__ x, const T* __restrict__ y, float* __restrict__ c, NArgs a) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const LoopNestCfg& L = a.n;
  if (t >= L.ext[0]) return;
  int64_t ox = t * L.dx[0], oy = t * L.dy[0], oc = t * L.dc[0];
  int64_t idx[kMaxLoopNest] = {0};
  int64_t total = 1;
  for (int l = 1; l < L.n; ++l) total *= L.ext[l];
  int64_t cur = oc;
  float acc = 0.f;
  for (int64_t it = 0; it < total; ++it) {
    if (oc != cur) {
      c[cur] += acc;
      acc = 0.f;
      cur = oc;
    }
    acc = fmaf(ldf(x, ox), ldf(y, oy), acc);
    // odometer over loops n-1 .. 1
    for (int l = L.n - 1; l >= 1; --l) {
      if (++idx[l] < L.ext[l]) { ox += L.dx[l]; oy += L.dy[l]; oc += L.dc[l]; break; }
      idx[l] = 0;
      ox -= L.dx[l] * (L.ext[l] - 1); oy -= L.dy[l] * (L.ext[l] - 1); oc -= L.dc[l] * (L.ext[l] - 1);
    }
    if (a.deadline && (it & 255) == 255 && gtimer() > *a.deadline) {
      atomicExch(a.timed_out, 1);
      return;
    }
  }
  c[cur] += acc;
}

// ---- K6 parity reducer -------------------------------------------------------
__global__ void parity_kernel(float* __restrict__ c, const double* __restrict__ ref, int64_t n, double rtol,
                              double atol, unsigned long long* slot, int poison) {
  double worst = 0.0;
  unsigned long long bad = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double r = ref[i], v = (double)c[i];
    double err = fabs(v - r);
    if (!(err <= atol + rtol * fabs(r))) ++bad;
    if (isnan(err)) err = INFINITY;
    worst = fmax(worst, err);
    if (poison) c[i] = __int_as_float(0x7fffffff);
  }
  for (int o = 16; o; o >>= 1) {
    worst = fmax(worst, __shfl_xor_sync(0xffffffffu, worst, o));
    bad += __shfl_xor_sync(0xffffffffu, bad, o);
  }
  // one pair of atomics per block (same-address atomics from every warp
  // serialise in L2 and dominated this kernel)
  __shared__ double s_worst[32];
  __shared__ unsigned long long s_bad[32];
  const int w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  if ((threadIdx.x & 31) == 0) { s_worst[w] = worst; s_bad[w] = bad; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 1; k < nw; ++k) { worst = fmax(worst, s_worst[k]); bad += s_bad[k]; }
    atomicMax(slot, (unsigned long long)__double_as_longlong(worst));
    if (bad) atomicAdd(slot + 1, bad);
  }
}

__global__ void arm_kernel(unsigned long long* s, const int* prev_flag, const unsigned long long* prev_parity,
                           double factor, unsigned long long floor_ns, unsigned long long cap_ns) {
  const unsigned long long now = gtimer();
  if (prev_flag && !*prev_flag && prev_parity[1] == 0) {
    // s[3]: end stamp of the previous candidate's kernels (launch_stamp), so
    // host enqueue gaps between candidates do not inflate the best time
    unsigned long long el = (s[3] > s[1] ? s[3] : now) - s[1];
    el = el > s[4] ? el - s[4] : 0;  // minus the calibrated empty-candidate overhead
    if (el < s[2]) s[2] = el;
  }
  unsigned long long t = cap_ns;
  if (factor > 0.0 && s[2] != ~0ull) {
    double want = factor * (double)s[2];
    t = want < (double)floor_ns ? floor_ns : (want > (double)cap_ns ? cap_ns : (unsigned long long)want);
  }
  s[0] = now + t;
  s[1] = now;
}

__global__ void stamp_kernel(unsigned long long* s) { s[3] = gtimer(); }

__global__ void delay_kernel(unsigned long long ns) {
  unsigned long long end = gtimer() + ns;
  while (gtimer() < end) {
  }
}

__global__ void to_bf16_kernel(const float* __restrict__ in, __nv_bfloat16* __restrict__ out, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = __float2bfloat16_rn(in[i]);
}

// out[b][c][r] = in[b][r][c]
__global__ void transpose_kernel(const __nv_bfloat16* __restrict__ in, __nv_bfloat16* __restrict__ out, int64_t rows,
                                 int64_t cols) {
  __shared__ __nv_bfloat16 tile[32][33];
  const int64_t b = blockIdx.z;
  const int64_t r0 = blockIdx.y * 32, c0 = blockIdx.x * 32;
  const __nv_bfloat16* src = in + b * rows * cols;
  __nv_bfloat16* dst = out + b * rows * cols;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    int64_t r = r0 + i, cc = c0 + threadIdx.x;
    if (r < rows && cc < cols) tile[i][threadIdx.x] = src[r * cols + cc];
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    int64_t cc = c0 + i, r = r0 + threadIdx.x;
    if (r < rows && cc < cols) dst[cc * rows + r] = tile[threadIdx.x][i];
  }
}

template <typename T, int RM, int RN>
cudaError_t simt_launch(const void* x, const void* y, float* c, const SArgs& a, dim3 grid, int threads, size_t smem,
                        cudaStream_t st) {
  auto fn = simt_gemm<T, RM, RN>;
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
  if (a.persist) {
    static int sms = 0;
    if (!sms) {
      int dev = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    }
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, threads, smem) != cudaSuccess || per_sm < 1) {
      cudaGetLastError();
      per_sm = 1;
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

}  // namespace
int opt_in_dynamic_smem(const void* fn);
namespace {

typedef cudaError_t (*SimtLauncher)(const void*, const void*, float*, const SArgs&, dim3, int, size_t, cudaStream_t);

template <typename T, int RM>
void fill_row(SimtLauncher* row) {
  row[0] = 1 * RM <= 64 ? simt_launch<T, RM, 1> : nullptr;
  row[1] = 2 * RM <= 64 ? simt_launch<T, RM, 2> : nullptr;
  row[2] = 3 * RM <= 64 ? simt_launch<T, RM, 3> : nullptr;
  row[3] = 4 * RM <= 64 ? simt_launch<T, RM, 4> : nullptr;
  row[4] = 6 * RM <= 64 ? simt_launch<T, RM, 6> : nullptr;
  row[5] = 8 * RM <= 64 ? simt_launch<T, RM, 8> : nullptr;
  row[6] = 12 * RM <= 64 ? simt_launch<T, RM, 12> : nullptr;
  row[7] = 16 * RM <= 64 ? simt_launch<T, RM, 16> : nullptr;
}

template <typename T>
struct SimtTable {
  SimtLauncher t[8][8];
  SimtTable() {
    fill_row<T, 1>(t[0]);
    fill_row<T, 2>(t[1]);
    fill_row<T, 3>(t[2]);
    fill_row<T, 4>(t[3]);
    fill_row<T, 6>(t[4]);
    fill_row<T, 8>(t[5]);
    fill_row<T, 12>(t[6]);
    fill_row<T, 16>(t[7]);
  }
};

}  // namespace

int opt_in_dynamic_smem(const void* fn) {
  int dev = 0, optin = 0;
  cudaFuncAttributes fa;
  if (cudaGetDevice(&dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess ||
      cudaFuncGetAttributes(&fa, fn) != cudaSuccess) {
    cudaGetLastError();
    return -1;
  }
  int dyn = optin - static_cast<int>(fa.sharedSizeBytes);
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn) != cudaSuccess) {
    cudaGetLastError();
    return -1;
  }
  return dyn;
}

namespace {

int grid_for(int64_t n, int threads) {
  int64_t g = (n + threads - 1) / threads;
  return (int)(g < 148 * 32 ? (g < 1 ? 1 : g) : 148 * 32);
}

}  // namespace

void launch_reference(const void* x, const void* y, double* out, const Strides& s, bool bf16, cudaStream_t st) {
  int64_t total = s.ext[0] * s.ext[1] * s.ext[2];
  int g = grid_for(total, 256);
  if (bf16)
    contract_naive<__nv_bfloat16, double, double><<<g, 256, 0, st>>>(
        static_cast<const __nv_bfloat16*>(x), static_cast<const __nv_bfloat16*>(y), out, s);
  else
    contract_naive<float, double, double><<<g, 256, 0, st>>>(static_cast<const float*>(x),
                                                             static_cast<const float*>(y), out, s);
}

void launch_naive(const void* x, const void* y, float* c, const Strides& s, bool bf16, cudaStream_t st) {
  int64_t total = s.ext[0] * s.ext[1] * s.ext[2];
  int g = (int)((total + 255) / 256);
  if (bf16)
    contract_naive<__nv_bfloat16, float, float><<<g, 256, 0, st>>>(
        static_cast<const __nv_bfloat16*>(x), static_cast<const __nv_bfloat16*>(y), c, s);
  else
    contract_naive<float, float, float><<<g, 256, 0, st>>>(static_cast<const float*>(x),
                                                           static_cast<const float*>(y), c, s);
}

// CUDA loads kernels lazily on first use; a first launch inside a checked
// (timed, deadline-armed) run would charge the module load to the candidate.
void preload_simt_kernels() {
  static SimtTable<float> tf;
  static SimtTable<__nv_bfloat16> tb;
  SArgs a{};
  for (int i = 0; i < 8; ++i)
    for (int j = 0; j < 8; ++j) {
      if (tf.t[i][j]) tf.t[i][j](nullptr, nullptr, nullptr, a, dim3(1), 1, static_cast<size_t>(-1), nullptr);
      if (tb.t[i][j]) tb.t[i][j](nullptr, nullptr, nullptr, a, dim3(1), 1, static_cast<size_t>(-1), nullptr);
    }
  cudaFuncAttributes at;
  cudaFuncGetAttributes(&at, parity_kernel);
  cudaFuncGetAttributes(&at, arm_kernel);
  cudaFuncGetAttributes(&at, stamp_kernel);
  cudaFuncGetAttributes(&at, contract_naive<__nv_bfloat16, float, float>);
  cudaFuncGetAttributes(&at, contract_naive<float, float, float>);
  cudaFuncGetAttributes(&at, loopnest_contract<__nv_bfloat16>);
  cudaFuncGetAttributes(&at, loopnest_contract<float>);
  cudaGetLastError();
}

bool launch_simt(const void* x, const void* y, float* c, const Strides& s, const SimtCfg& cfg, bool bf16,
                 const unsigned long long* deadline, int* timed_out, cudaStream_t st) {
  static SimtTable<float> tf;
  static SimtTable<__nv_bfloat16> tb;
  int i = simt_tile_index(cfg.rm), j = simt_tile_index(cfg.rn);
  if (i < 0 || j < 0) return false;
  SimtLauncher fn = bf16 ? tb.t[i][j] : tf.t[i][j];
  if (!fn) return false;
  SArgs a;
  a.s = s;
  a.tb = cfg.tb; a.tm = cfg.tm; a.tn = cfg.tn; a.rb = cfg.rb; a.bk = cfg.bk; a.kt = cfg.kt;
  a.deadline = deadline;
  a.timed_out = timed_out;
  static const bool no_persist = getenv("LSB_SIMT_NOPERSIST") && atoi(getenv("LSB_SIMT_NOPERSIST")) != 0;
  a.persist = deadline && !no_persist ? 1 : 0;
  a.ntn = a.ntm = a.ntb = 1;
  const int64_t bm = cfg.tm * cfg.rm, bn = cfg.tn * cfg.rn;
  const int vw = bf16 ? 8 : 4;
  // operand X (rows = M): contiguous along k or m?
  a.x_kfast = s.sx[3] == 1 || s.sx[1] != 1;
  a.y_kfast = s.sy[3] == 1 || s.sy[2] != 1;
  auto vec_ok = [&](bool kfast, int64_t s_b, int64_t s_r, int64_t s_k, int64_t nr) {
    if (kfast) return s_k == 1 && cfg.bk % vw == 0 && s_r % vw == 0 && s_b % vw == 0;
    return s_r == 1 && nr % vw == 0 && s_k % vw == 0 && s_b % vw == 0;
  };
  a.va = vec_ok(a.x_kfast, s.sx[0], s.sx[1], s.sx[3], bm) ? vw : 1;
  a.vb = vec_ok(a.y_kfast, s.sy[0], s.sy[2], s.sy[3], bn) ? vw : 1;
  // k-fast staging writes columns of S[kk][r]: pad rows by one word to spread
  // banks; r-fast staging writes rows and keeps 16-byte alignment for reads
  a.lda = (int)(a.x_kfast ? bm + 1 : bm);
  a.ldb = (int)(a.y_kfast ? bn + 1 : bn);
  a.a_vec_smem = (a.lda % 4 == 0) && (cfg.rm % 4 == 0);
  a.b_vec_smem = (a.ldb % 4 == 0) && (cfg.rn % 4 == 0);
  a.c_vec = s.sc[2] == 1 && cfg.rn % 4 == 0 && s.sc[1] % 4 == 0 && s.sc[0] % 4 == 0;
  const size_t a_words = ((size_t)cfg.tb * cfg.bk * a.lda + 3) & ~(size_t)3;
  size_t smem = (a_words + (size_t)cfg.tb * cfg.bk * a.ldb) * sizeof(float);
  // fp32 with more than one k-tile: double-buffer through cp.async when two
  // tile sets fit (the hardware validator judged the single set)
  static int db_max = -1;
  if (db_max < 0) {
    int dev = 0, v = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    db_max = v - 2048;
  }
  static const bool no_db = getenv("LSB_SIMT_NODB") && atoi(getenv("LSB_SIMT_NODB")) != 0;
  const size_t set_words = (a_words + (size_t)cfg.tb * cfg.bk * a.ldb + 3) & ~(size_t)3;
  a.db = !bf16 && !no_db && cfg.kt > 1 && 2 * set_words * sizeof(float) <= static_cast<size_t>(db_max) ? 1 : 0;
  if (a.db) smem = 2 * set_words * sizeof(float);
  dim3 grid((unsigned)cfg.gn, (unsigned)cfg.gm, (unsigned)cfg.gb);
  return fn(x, y, c, a, grid, (int)(cfg.tb * cfg.tm * cfg.tn), smem, st) == cudaSuccess;
}

void launch_loopnest(const void* x, const void* y, float* c, const LoopNestCfg& cfg, bool bf16,
                     const unsigned long long* deadline, int* timed_out, cudaStream_t st) {
  NArgs a;
  a.n = cfg;
  a.deadline = deadline;
  a.timed_out = timed_out;
  int threads = 128;
  int g = (int)((cfg.ext[0] + threads - 1) / threads);
  if (bf16)
    loopnest_contract<__nv_bfloat16><<<g, threads, 0, st>>>(static_cast<const __nv_bfloat16*>(x),
                                                            static_cast<const __nv_bfloat16*>(y), c, a);
  else
    loopnest_contract<float><<<g, threads, 0, st>>>(static_cast<const float*>(x), static_cast<const float*>(y), c, a);
}

void launch_parity(float* c, const double* ref, int64_t n, double rtol, double atol, unsigned long long* slot,
                   bool poison, cudaStream_t st) {
  int64_t g = (n + 511) / 512;  // >= 2 elements per thread, at most 2 blocks per SM
  if (g > 296) g = 296;
  if (g < 1) g = 1;
  parity_kernel<<<(unsigned)g, 256, 0, st>>>(c, ref, n, rtol, atol, slot, poison ? 1 : 0);
}

void launch_arm(unsigned long long* state, const int* prev_flag, const unsigned long long* prev_parity,
                double factor, unsigned long long floor_ns, unsigned long long cap_ns, cudaStream_t st) {
  arm_kernel<<<1, 1, 0, st>>>(state, prev_flag, prev_parity, factor, floor_ns, cap_ns);
}

void launch_delay(unsigned long long ns, cudaStream_t st) { delay_kernel<<<1, 1, 0, st>>>(ns); }

void launch_stamp(unsigned long long* state, cudaStream_t st) { stamp_kernel<<<1, 1, 0, st>>>(state); }

void launch_to_bf16(const float* in, __nv_bfloat16* out, int64_t n, cudaStream_t st) {
  to_bf16_kernel<<<grid_for(n, 256), 256, 0, st>>>(in, out, n);
}

void launch_transpose_bf16(const __nv_bfloat16* in, __nv_bfloat16* out, int64_t batch, int64_t rows, int64_t cols,
                           cudaStream_t st) {
  dim3 grid((unsigned)((cols + 31) / 32), (unsigned)((rows + 31) / 32), (unsigned)batch);
  transpose_kernel<<<grid, dim3(32, 8), 0, st>>>(in, out, rows, cols);
}

}  // namespace lsb
