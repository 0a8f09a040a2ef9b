// Generic block executor kernel (see generic.hpp).
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "generic.cuh"

namespace lsb {

namespace {

constexpr int kStack = 32;

__device__ __forceinline__ double gload(const GenBuffers& B, int buf, const int64_t* idx, int nd) {
  int64_t off = 0;
  for (int d = 0; d < nd; ++d) {
    const int64_t e = B.shape[buf][d];
    if (idx[d] < 0 || idx[d] >= e) return 0.0;  // untaken Select branch (pad guard)
    off = off * e + idx[d];
  }
  switch (B.dtype[buf]) {
    case 0: return (double)__bfloat162float(static_cast<const __nv_bfloat16*>(B.ptr[buf])[off]);
    case 1: return (double)static_cast<const float*>(B.ptr[buf])[off];
    default: return static_cast<const double*>(B.ptr[buf])[off];
  }
}

__device__ __forceinline__ void gstore(const GenBuffers& B, int buf, const int64_t* idx, int nd, double v) {
  int64_t off = 0;
  for (int d = 0; d < nd; ++d) off = off * B.shape[buf][d] + idx[d];
  switch (B.dtype[buf]) {
    case 0: static_cast<__nv_bfloat16*>(B.ptr[buf])[off] = __float2bfloat16_rn((float)v); break;
    case 1: static_cast<float*>(B.ptr[buf])[off] = (float)v; break;
    default: static_cast<double*>(B.ptr[buf])[off] = v; break;
  }
}

__device__ double geval(const int64_t* code, const double* vars, const GenBuffers& B) {
  double st[kStack];
  int sp = 0;
  const int64_t n = code[0];
  for (int64_t i = 0; i < n; ++i) {
    const int64_t op = code[1 + 2 * i], arg = code[2 + 2 * i];
    switch (op) {
      case G_CONST: st[sp++] = (double)arg; break;
      case G_VAR: st[sp++] = vars[arg]; break;
      case G_LOAD: {
        const int buf = (int)(arg & 0xffffffff), nd = (int)(arg >> 32);
        int64_t idx[8];
        for (int d = nd - 1; d >= 0; --d) idx[d] = (int64_t)st[--sp];
        st[sp++] = gload(B, buf, idx, nd);
        break;
      }
      case G_SEL: {
        double o = st[--sp], t = st[--sp], c = st[--sp];
        st[sp++] = c != 0.0 ? t : o;
        break;
      }
      default: {
        double b = st[--sp], a = st[--sp], r = 0.0;
        switch (op) {
          case G_ADD: r = a + b; break;
          case G_SUB: r = a - b; break;
          case G_MUL: r = a * b; break;
          case G_MAX: r = fmax(a, b); break;
          case G_MIN: r = fmin(a, b); break;
          case G_FDIV: r = floor(a / b); break;
          case G_MOD: r = a - b * floor(a / b); break;
        }
        st[sp++] = r;
      }
    }
  }
  return st[0];
}

// Acc: the accumulation type (float for candidates, double for the reference)
template <typename Acc>
__global__ void generic_block_kernel(GenBlock g, const int64_t* __restrict__ code, GenBuffers B,
                                     const unsigned long long* deadline, int* timed_out) {
  double vars[kGenMaxLoops];
  int visited = 0;
  for (int64_t pt = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; pt < g.points;
       pt += (int64_t)gridDim.x * blockDim.x) {
    // elementwise stages have no reduction loop to check in: look at the
    // clock every 16 points (one interpreted point costs ~1 us)
    if (deadline && (++visited & 15) == 0) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (t > *deadline) { atomicExch(timed_out, 1); return; }
    }
    // decode the point loops (nest order, last fastest); reduction loops start at 0
    int64_t rem = pt;
    for (int i = g.nl - 1; i >= 0; --i) {
      if ((g.red_mask >> i) & 1u) { vars[i] = 0.0; continue; }
      vars[i] = (double)(rem % g.ext[i]);
      rem /= g.ext[i];
    }
    int64_t sidx[8];
    for (int d = 0; d < g.store_ndim; ++d) sidx[d] = (int64_t)geval(code + g.store_code[d], vars, B);
    if (g.init_code < 0) {
      gstore(B, g.store_buf, sidx, g.store_ndim, geval(code + g.value_code, vars, B));
      continue;
    }
    Acc acc = (Acc)geval(code + g.init_code, vars, B);
    for (int64_t it = 0; it < g.red_trip; ++it) {
      acc += (Acc)geval(code + g.value_code, vars, B);
      for (int i = g.nl - 1; i >= 0; --i) {  // odometer over the reduction loops
        if (!((g.red_mask >> i) & 1u)) continue;
        if (vars[i] + 1.0 < (double)g.ext[i]) { vars[i] += 1.0; break; }
        vars[i] = 0.0;
      }
      if (deadline && (it & 7) == 7) {  // bytecode iterations are slow: check often
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if (t > *deadline) { atomicExch(timed_out, 1); return; }
      }
    }
    gstore(B, g.store_buf, sidx, g.store_ndim, (double)acc);
    if (g.epi_code >= 0) {
      // last reduction iteration: every reduction var at extent-1
      for (int i = 0; i < g.nl; ++i)
        if ((g.red_mask >> i) & 1u) vars[i] = (double)(g.ext[i] - 1);
      gstore(B, g.store_buf, sidx, g.store_ndim, geval(code + g.epi_code, vars, B));
    }
  }
}

// PVU-faithful variant: thread t owns iteration t of the outermost loop (the
// parallel one); every other loop runs in nest order inside the thread, with
// the reference's statement semantics per iteration (init on the first
// reduction iteration, accumulate in place, epilogue on the last).
template <typename Acc>
__global__ void generic_nest_kernel(GenBlock g, const int64_t* __restrict__ code, GenBuffers B,
                                    const unsigned long long* deadline, int* timed_out) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= g.ext[0]) return;
  double vars[kGenMaxLoops];
  vars[0] = (double)t;
  int64_t inner = 1;
  for (int i = 1; i < g.nl; ++i) { vars[i] = 0.0; inner *= g.ext[i]; }
  int64_t sidx[8];
  for (int64_t it = 0; it < inner; ++it) {
    for (int d = 0; d < g.store_ndim; ++d) sidx[d] = (int64_t)geval(code + g.store_code[d], vars, B);
    if (g.init_code < 0) {
      gstore(B, g.store_buf, sidx, g.store_ndim, geval(code + g.value_code, vars, B));
    } else {
      bool first = true, last = true;
      for (int i = 0; i < g.nl; ++i)
        if ((g.red_mask >> i) & 1u) {
          first &= vars[i] == 0.0;
          last &= vars[i] == (double)(g.ext[i] - 1);
        }
      Acc acc = first ? (Acc)geval(code + g.init_code, vars, B) : (Acc)gload(B, g.store_buf, sidx, g.store_ndim);
      acc += (Acc)geval(code + g.value_code, vars, B);
      gstore(B, g.store_buf, sidx, g.store_ndim, (double)acc);
      if (last && g.epi_code >= 0) gstore(B, g.store_buf, sidx, g.store_ndim, geval(code + g.epi_code, vars, B));
    }
    for (int i = g.nl - 1; i >= 1; --i) {
      if (vars[i] + 1.0 < (double)g.ext[i]) { vars[i] += 1.0; break; }
      vars[i] = 0.0;
    }
    if (deadline) {  // one interpreted iteration costs ~1-10 us: check every one
      unsigned long long now;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
      if (now > *deadline) { atomicExch(timed_out, 1); return; }
    }
  }
}

// AFFCOPY: thread per point of the block's loops (nest order, last fastest)
// 32-bit arithmetic throughout (every index and offset of a runner buffer
// fits; the planner checks the buffer sizes): 64-bit division is a long
// instruction sequence and was the kernel's bottleneck
__device__ __forceinline__ int32_t qsum(const QSum& q, const uint32_t* lv) {
  int32_t acc = static_cast<int32_t>(q.c0);
  for (int i = 0; i < q.n; ++i) {
    const QTerm& t = q.t[i];
    uint32_t x = lv[t.loop];
    if (t.div > 1) x /= static_cast<uint32_t>(t.div);
    if (t.mod) x %= static_cast<uint32_t>(t.mod);
    acc += static_cast<int32_t>(x) * static_cast<int32_t>(t.coef);
  }
  return acc;
}

template <typename Ti, typename To>
__global__ void affcopy_kernel(const __grid_constant__ CopyCfg c, const Ti* __restrict__ in, To* __restrict__ out,
                               const unsigned long long* deadline, int* timed_out) {
  // thread unit: `vec` consecutive elements of the contiguous innermost run
  const uint32_t vec = static_cast<uint32_t>(c.vec);
  const uint32_t units = static_cast<uint32_t>(c.points / c.vec);
  const int outer = c.nl - c.run_loops;
  int visited = 0;
  for (uint32_t u = blockIdx.x * blockDim.x + threadIdx.x; u < units; u += gridDim.x * blockDim.x) {
    // a stage the schedule recomputes redundantly (compute_at inside loops
    // it does not index) can be huge: checked launches look at the clock
    if (deadline && (++visited & 15) == 0) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (t > *deadline) { atomicExch(timed_out, 1); return; }
    }
    uint32_t lv[kCopyMaxLoops];
    // digits of the run loops come from the element index inside the run
    const uint32_t per_run = static_cast<uint32_t>(c.run) / vec;
    uint32_t rem = u / per_run;
    uint32_t e0 = (u - rem * per_run) * vec;
    for (int l = c.nl - 1; l >= outer; --l) {
      const uint32_t e = static_cast<uint32_t>(c.ext[l]);
      const uint32_t q = e0 / e;
      lv[l] = e0 - q * e;
      e0 = q;
    }
    for (int l = outer - 1; l >= 0; --l) {
      const uint32_t e = static_cast<uint32_t>(c.ext[l]);
      const uint32_t q = rem / e;
      lv[l] = rem - q * e;
      rem = q;
    }
    bool inb = true;
    for (int d = 0; d < c.ng; ++d) {
      const int32_t x = qsum(c.g[d], lv);
      inb &= x >= 0 && x < static_cast<int32_t>(c.gext[d]);
    }
    const int32_t i0 = qsum(c.in, lv), o0 = qsum(c.out, lv);
    for (uint32_t k = 0; k < vec; ++k) {
      float v = 0.f;
      if (inb) {
        if constexpr (sizeof(Ti) == 2) v = __bfloat162float(in[i0 + k]);
        else v = static_cast<float>(in[i0 + k]);
      }
      if constexpr (sizeof(To) == 2) out[o0 + k] = __float2bfloat16_rn(v);
      else out[o0 + k] = v;
    }
  }
}

}  // namespace

void preload_generic_kernels() {
  cudaFuncAttributes at;
  cudaFuncGetAttributes(&at, affcopy_kernel<__nv_bfloat16, __nv_bfloat16>);  // (also preloads the others below)
  cudaFuncGetAttributes(&at, affcopy_kernel<__nv_bfloat16, float>);
  cudaFuncGetAttributes(&at, affcopy_kernel<float, __nv_bfloat16>);
  cudaFuncGetAttributes(&at, affcopy_kernel<float, float>);
  cudaFuncGetAttributes(&at, generic_block_kernel<float>);
  cudaFuncGetAttributes(&at, generic_block_kernel<double>);
  cudaFuncGetAttributes(&at, generic_nest_kernel<float>);
  cudaGetLastError();
}

bool launch_affcopy(const CopyCfg& c, const GenBuffers& B, const unsigned long long* deadline, int* timed_out,
                    cudaStream_t st) {
  const int ti = B.dtype[c.in_buf], to = B.dtype[c.out_buf];
  if (ti > 1 || to > 1) return false;
  const int threads = 256;
  int64_t blocks = (c.points / c.vec + threads - 1) / threads;
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (blocks < 1) blocks = 1;
  const void* in = B.ptr[c.in_buf];
  void* out = B.ptr[c.out_buf];
  const unsigned nb = static_cast<unsigned>(blocks);
  if (ti == 0 && to == 0)
    affcopy_kernel<__nv_bfloat16, __nv_bfloat16><<<nb, threads, 0, st>>>(c, static_cast<const __nv_bfloat16*>(in),
                                                                        static_cast<__nv_bfloat16*>(out), deadline, timed_out);
  else if (ti == 0)
    affcopy_kernel<__nv_bfloat16, float><<<nb, threads, 0, st>>>(c, static_cast<const __nv_bfloat16*>(in),
                                                                static_cast<float*>(out), deadline, timed_out);
  else if (to == 0)
    affcopy_kernel<float, __nv_bfloat16><<<nb, threads, 0, st>>>(c, static_cast<const float*>(in),
                                                                static_cast<__nv_bfloat16*>(out), deadline, timed_out);
  else
    affcopy_kernel<float, float><<<nb, threads, 0, st>>>(c, static_cast<const float*>(in), static_cast<float*>(out), deadline, timed_out);
  return cudaGetLastError() == cudaSuccess;
}

bool launch_generic_nest(const GenBlock& g, const int64_t* code, const GenBuffers& B,
                         const unsigned long long* deadline, int* timed_out, cudaStream_t st) {
  int threads = 128;
  int64_t blocks = (g.ext[0] + threads - 1) / threads;
  if (blocks < 1) blocks = 1;
  generic_nest_kernel<float><<<(unsigned)blocks, threads, 0, st>>>(g, code, B, deadline, timed_out);
  return cudaGetLastError() == cudaSuccess;
}

bool launch_generic_block(const GenBlock& g, const int64_t* code, const GenBuffers& B, bool fp64,
                          const unsigned long long* deadline, int* timed_out, cudaStream_t st) {
  int threads = 128;
  int64_t blocks = (g.points + threads - 1) / threads;
  if (blocks > 148 * 64) blocks = 148 * 64;
  if (blocks < 1) blocks = 1;
  if (fp64)
    generic_block_kernel<double><<<(unsigned)blocks, threads, 0, st>>>(g, code, B, deadline, timed_out);
  else
    generic_block_kernel<float><<<(unsigned)blocks, threads, 0, st>>>(g, code, B, deadline, timed_out);
  return cudaGetLastError() == cudaSuccess;
}

}  // namespace lsb
