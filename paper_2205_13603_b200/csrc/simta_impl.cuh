// SIMT-A: affine SIMT tile kernel for multi-axis contractions (implicit GEMM).
// Included by simta_f32.cu / simta_bf16.cu (one dtype each, compiled in
// parallel).  See affine.hpp for the mapping convention.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "affine.hpp"
#include "simta.cuh"

namespace lsb {
namespace simta {

__device__ __forceinline__ float ld1(const float* p, int64_t i) { return __ldg(p + i); }
__device__ __forceinline__ float ld1(const __nv_bfloat16* p, int64_t i) { return __bfloat162float(p[i]); }

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// digits of idx over the parts of one list (nest order, last fastest); the
// indices and extents fit in 32 bits, and 32-bit division is ~4x cheaper
__device__ __forceinline__ void decode(const AList& L, int64_t idx64, int64_t* sx, int64_t* sy, int64_t* sc,
                                       int64_t* g0, int64_t* g1) {
  uint32_t idx = static_cast<uint32_t>(idx64);
  for (int p = L.n - 1; p >= 0; --p) {
    const uint32_t e = static_cast<uint32_t>(L.ext[p]);
    const uint32_t q = idx / e;
    const int64_t d = static_cast<int64_t>(idx - q * e);
    idx = q;
    *sx += d * L.cx[p];
    *sy += d * L.cy[p];
    *sc += d * L.cc[p];
    *g0 += d * L.cg0[p];
    *g1 += d * L.cg1[p];
  }
}

template <typename T, int RM, int RN>
__global__ void __launch_bounds__(1024) simta_kernel(const T* __restrict__ x, const T* __restrict__ y,
                                                     float* __restrict__ c, SimtaArgs a) {
  extern __shared__ float sm[];
  __shared__ int abort_flag;
  const int tid = threadIdx.x;
  const int tn = (int)a.tn, tm = (int)a.tm, nthr = tm * tn;
  const int tn_i = tid % tn, tm_i = tid / tn;
  const int bm = tm * RM, bn = tn * RN, bk = (int)a.bk;
  const int lda = bm + 1, ldb = bn + 1;
  float* As = sm;
  float* Bs = As + bk * lda;
  int* offXM = reinterpret_cast<int*>(Bs + bk * ldb);
  int* offCM = offXM + bm;
  int* offYN = offCM + bm;
  int* offCN = offYN + bn;
  int* offXK = offCN + bn;
  int* offYK = offXK + bk;
  int* gM0 = offYK + bk;
  int* gM1 = gM0 + bm;
  int* gK0 = gM1 + bm;
  int* gK1 = gK0 + bk;

  // ---- per-CTA address tables ----
  for (int mm = tid; mm < bm; mm += nthr) {
    int64_t sx = 0, sy = 0, sc = 0, g0 = 0, g1 = 0;
    decode(a.m_thr, mm / RM, &sx, &sy, &sc, &g0, &g1);
    decode(a.m_reg, mm % RM, &sx, &sy, &sc, &g0, &g1);
    offXM[mm] = (int)sx; offCM[mm] = (int)sc; gM0[mm] = (int)g0; gM1[mm] = (int)g1;
  }
  for (int nn = tid; nn < bn; nn += nthr) {
    int64_t sx = 0, sy = 0, sc = 0, g0 = 0, g1 = 0;
    decode(a.n_thr, nn / RN, &sx, &sy, &sc, &g0, &g1);
    decode(a.n_reg, nn % RN, &sx, &sy, &sc, &g0, &g1);
    offYN[nn] = (int)sy; offCN[nn] = (int)sc;
  }
  for (int kk = tid; kk < bk; kk += nthr) {
    int64_t sx = 0, sy = 0, sc = 0, g0 = 0, g1 = 0;
    decode(a.k_bk, kk, &sx, &sy, &sc, &g0, &g1);
    offXK[kk] = (int)sx; offYK[kk] = (int)sy; gK0[kk] = (int)g0; gK1[kk] = (int)g1;
  }
  const int64_t ntiles = a.persist ? a.ntn * a.ntm : 1;
  for (int64_t tile = a.persist ? blockIdx.x : 0; tile < ntiles; tile += a.persist ? gridDim.x : 1) {
  int64_t bx = a.x0, by = a.y0, bc = a.c0, bg0 = a.g0[0], bg1 = a.g0[1];
  decode(a.m_grid, a.persist ? tile / a.ntn : blockIdx.y, &bx, &by, &bc, &bg0, &bg1);
  decode(a.n_grid, a.persist ? tile % a.ntn : blockIdx.x, &bx, &by, &bc, &bg0, &bg1);
  __syncthreads();

  float acc[RM][RN];
#pragma unroll
  for (int i = 0; i < RM; ++i)
#pragma unroll
    for (int j = 0; j < RN; ++j) acc[i][j] = 0.f;

  for (int64_t kt = 0; kt < a.kt; ++kt) {
    if (a.deadline) {
      if (tid == 0) abort_flag = gtimer() > *a.deadline;
      __syncthreads();
      if (abort_flag) {
        if (tid == 0) atomicExch(a.timed_out, 1);
        return;
      }
    }
    int64_t kx = bx, ky = by, kc = 0, kg0 = bg0, kg1 = bg1;
    decode(a.k_tile, kt, &kx, &ky, &kc, &kg0, &kg1);
    // A tile, k fastest (consecutive threads walk the contiguous ci axis);
    // carried (mm, kk) indices: no per-element division
    {
      int kk = tid % bk, mm = tid / bk;
      const int skk = nthr % bk, smm = nthr / bk;
      for (int e = tid; e < bm * bk; e += nthr) {
        float v = 0.f;
        bool ok = true;
        if (a.ng > 0) {
          const int64_t h = kg0 + gM0[mm] + gK0[kk];
          ok = h >= 0 && h < a.gext[0];
          if (a.ng > 1) {
            const int64_t w2 = kg1 + gM1[mm] + gK1[kk];
            ok = ok && w2 >= 0 && w2 < a.gext[1];
          }
        }
        if (ok) v = ld1(x, kx + offXM[mm] + offXK[kk]);
        As[kk * lda + mm] = v;
        kk += skk;
        mm += smm;
        if (kk >= bk) { kk -= bk; ++mm; }
      }
    }
    // B tile, n fastest (co is contiguous in HWIO weights)
    {
      int nn = tid % bn, kk = tid / bn;
      const int snn = nthr % bn, skk = nthr / bn;
      for (int e = tid; e < bn * bk; e += nthr) {
        Bs[kk * ldb + nn] = ld1(y, ky + offYN[nn] + offYK[kk]);
        nn += snn;
        kk += skk;
        if (nn >= bn) { nn -= bn; ++kk; }
      }
    }
    __syncthreads();
    const float* Ap = As + tm_i * RM;
    const float* Bp = Bs + tn_i * RN;
    // checked launches look at the clock between 64-step chunks (see simt_gemm)
    const unsigned long long dlv = a.deadline ? *a.deadline : 0ull;
    for (int kc = 0; kc < bk; kc += 64) {
    if (a.deadline && kc && gtimer() > dlv) break;
    const int kend = min(bk, kc + 64);
#pragma unroll 4
    for (int kk = kc; kk < kend; ++kk) {
      float av[RM], bv[RN];
#pragma unroll
      for (int i = 0; i < RM; ++i) av[i] = Ap[kk * lda + i];
#pragma unroll
      for (int j = 0; j < RN; ++j) bv[j] = Bp[kk * ldb + j];
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
#pragma unroll
  for (int i = 0; i < RM; ++i)
#pragma unroll
    for (int j = 0; j < RN; ++j) c[bc + offCM[tm_i * RM + i] + offCN[tn_i * RN + j]] = acc[i][j];
  }  // tile loop
}

template <typename T, int RM, int RN>
cudaError_t launch_one(const void* x, const void* y, float* c, const SimtaArgs& a, size_t smem, cudaStream_t st) {
  auto fn = simta_kernel<T, RM, RN>;
  if (smem == static_cast<size_t>(-1)) {  // preload (see kernels.cu preload_simt_kernels)
    cudaFuncAttributes at;
    return cudaFuncGetAttributes(&at, fn);
  }
  static int max_dyn = -1;
  if (max_dyn < 0) {
    max_dyn = opt_in_dynamic_smem(reinterpret_cast<const void*>(fn));
    if (max_dyn <= 0) return cudaErrorInvalidValue;
  }
  if (smem > static_cast<size_t>(max_dyn)) return cudaErrorInvalidValue;
  const int threads = static_cast<int>(a.tm * a.tn);
  if (a.persist) {
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
    const int64_t wave = static_cast<int64_t>(sms) * per_sm;
    if (a.gn * a.gm > wave) {
      SimtaArgs p = a;
      p.ntn = a.gn;
      p.ntm = a.gm;
      fn<<<dim3(static_cast<unsigned>(wave)), threads, smem, st>>>(static_cast<const T*>(x),
                                                                   static_cast<const T*>(y), c, p);
      return cudaGetLastError();
    }
  }
  SimtaArgs p = a;
  p.persist = 0;
  dim3 grid(static_cast<unsigned>(a.gn), static_cast<unsigned>(a.gm), 1);
  fn<<<grid, threads, smem, st>>>(static_cast<const T*>(x), static_cast<const T*>(y), c, p);
  return cudaGetLastError();
}

typedef cudaError_t (*Launcher)(const void*, const void*, float*, const SimtaArgs&, size_t, cudaStream_t);

template <typename T, int RM>
void row(Launcher* r) {
  r[0] = launch_one<T, RM, 1>;
  r[1] = launch_one<T, RM, 2>;
  r[2] = RM * 3 <= 64 ? launch_one<T, RM, 3> : nullptr;
  r[3] = RM * 4 <= 64 ? launch_one<T, RM, 4> : nullptr;
  r[4] = RM * 6 <= 64 ? launch_one<T, RM, 6> : nullptr;
  r[5] = RM * 7 <= 64 ? launch_one<T, RM, 7> : nullptr;
  r[6] = RM * 8 <= 64 ? launch_one<T, RM, 8> : nullptr;
  r[7] = RM * 12 <= 64 ? launch_one<T, RM, 12> : nullptr;
  r[8] = RM * 14 <= 64 ? launch_one<T, RM, 14> : nullptr;
  r[9] = RM * 16 <= 64 ? launch_one<T, RM, 16> : nullptr;
}

template <typename T>
struct Table {
  Launcher t[10][10];
  Table() {
    row<T, 1>(t[0]); row<T, 2>(t[1]); row<T, 3>(t[2]); row<T, 4>(t[3]); row<T, 6>(t[4]);
    row<T, 7>(t[5]); row<T, 8>(t[6]); row<T, 12>(t[7]); row<T, 14>(t[8]); row<T, 16>(t[9]);
  }
};

template <typename T>
void preload_table() {
  static Table<T> t;
  SimtaArgs a{};
  for (int i = 0; i < 10; ++i)
    for (int j = 0; j < 10; ++j)
      if (t.t[i][j]) t.t[i][j](nullptr, nullptr, nullptr, a, static_cast<size_t>(-1), nullptr);
  cudaGetLastError();
}

}  // namespace simta
}  // namespace lsb
