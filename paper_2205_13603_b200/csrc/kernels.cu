// Runner kernels: reference output, NAIVE / SIMT / LOOPNEST candidate
// families, K6 parity reducer and timing utilities.  The tcgen05 family lives
// in tc_gemm.cu.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

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
template <typename T, int RM, int RN>
__global__ void __launch_bounds__(1024) simt_gemm(const T* __restrict__ x, const T* __restrict__ y,
                                                  float* __restrict__ c, SArgs a) {
  extern __shared__ float sm[];
  __shared__ int abort_flag;
  const int tid = threadIdx.x;
  const int nthr = (int)(a.tb * a.tm * a.tn);
  const int tn_i = tid % (int)a.tn;
  const int tm_i = (tid / (int)a.tn) % (int)a.tm;
  const int tb_i = tid / (int)(a.tn * a.tm);
  const int bm = (int)a.tm * RM, bn = (int)a.tn * RN, bk = (int)a.bk;
  float* As = sm;
  float* Bs = sm + a.tb * bk * bm;
  const int64_t m0 = (int64_t)blockIdx.y * bm, n0 = (int64_t)blockIdx.x * bn;
  const int64_t b0 = (int64_t)blockIdx.z * a.tb * a.rb;
  const Strides& s = a.s;
  const int a_total = (int)a.tb * bm * bk, b_total = (int)a.tb * bn * bk;

  for (int64_t rbi = 0; rbi < a.rb; ++rbi) {
    float acc[RM][RN];
#pragma unroll
    for (int i = 0; i < RM; ++i)
#pragma unroll
      for (int j = 0; j < RN; ++j) acc[i][j] = 0.f;

    for (int64_t kti = 0; kti < a.kt; ++kti) {
      if (a.deadline) {
        if (tid == 0) abort_flag = gtimer() > *a.deadline;
        __syncthreads();
        if (abort_flag) {
          if (tid == 0) atomicExch(a.timed_out, 1);
          return;
        }
      }
      const int64_t k0 = kti * bk;
      for (int e = tid; e < a_total; e += nthr) {
        int kk, mm, tbx;
        if (a.x_kfast) { kk = e % bk; int r = e / bk; mm = r % bm; tbx = r / bm; }
        else { mm = e % bm; int r = e / bm; kk = r % bk; tbx = r / bk; }
        const int64_t b = b0 + tbx * a.rb + rbi;
        As[(tbx * bk + kk) * bm + mm] = ldf(x, b * s.sx[0] + (m0 + mm) * s.sx[1] + (k0 + kk) * s.sx[3]);
      }
      for (int e = tid; e < b_total; e += nthr) {
        int kk, nn, tbx;
        if (a.y_kfast) { kk = e % bk; int r = e / bk; nn = r % bn; tbx = r / bn; }
        else { nn = e % bn; int r = e / bn; kk = r % bk; tbx = r / bk; }
        const int64_t b = b0 + tbx * a.rb + rbi;
        Bs[(tbx * bk + kk) * bn + nn] = ldf(y, b * s.sy[0] + (n0 + nn) * s.sy[2] + (k0 + kk) * s.sy[3]);
      }
      __syncthreads();
      const float* Ap = As + (int64_t)tb_i * bk * bm + tm_i * RM;
      const float* Bp = Bs + (int64_t)tb_i * bk * bn + tn_i * RN;
      for (int kk = 0; kk < bk; ++kk) {
        float av[RM], bv[RN];
#pragma unroll
        for (int i = 0; i < RM; ++i) av[i] = Ap[kk * bm + i];
#pragma unroll
        for (int j = 0; j < RN; ++j) bv[j] = Bp[kk * bn + j];
#pragma unroll
        for (int i = 0; i < RM; ++i)
#pragma unroll
          for (int j = 0; j < RN; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
      }
      __syncthreads();
    }
    const int64_t b = b0 + tb_i * a.rb + rbi;
#pragma unroll
    for (int i = 0; i < RM; ++i)
#pragma unroll
      for (int j = 0; j < RN; ++j)
        c[b * s.sc[0] + (m0 + tm_i * RM + i) * s.sc[1] + (n0 + tn_i * RN + j) * s.sc[2]] = acc[i][j];
  }
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
    if (a.deadline && (it & 4095) == 4095 && gtimer() > *a.deadline) {
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
  if ((threadIdx.x & 31) == 0) {
    atomicMax(slot, (unsigned long long)__double_as_longlong(worst));
    if (bad) atomicAdd(slot + 1, bad);
  }
}

__global__ void arm_kernel(unsigned long long* s, const int* prev_flag, const unsigned long long* prev_parity,
                           double factor, unsigned long long floor_ns, unsigned long long cap_ns) {
  const unsigned long long now = gtimer();
  if (prev_flag && !*prev_flag && prev_parity[1] == 0) {
    unsigned long long el = now - s[1];
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
  static int max_dyn = -1;  // per instantiation: opt-in limit minus the kernel's static smem
  if (max_dyn < 0) {
    max_dyn = opt_in_dynamic_smem(reinterpret_cast<const void*>(fn));
    if (max_dyn <= 0) return cudaErrorInvalidValue;
  }
  if (smem > static_cast<size_t>(max_dyn)) return cudaErrorInvalidValue;
  fn<<<grid, threads, smem, st>>>(static_cast<const T*>(x), static_cast<const T*>(y), c, a);
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
  a.x_kfast = s.sx[3] == 1;
  a.y_kfast = s.sy[3] == 1;
  a.deadline = deadline;
  a.timed_out = timed_out;
  dim3 grid((unsigned)cfg.gn, (unsigned)cfg.gm, (unsigned)cfg.gb);
  return fn(x, y, c, a, grid, (int)(cfg.tb * cfg.tm * cfg.tn), (size_t)cfg.smem_bytes, st) == cudaSuccess;
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
  parity_kernel<<<grid_for(n, 256), 256, 0, st>>>(c, ref, n, rtol, atol, slot, poison ? 1 : 0);
}

void launch_arm(unsigned long long* state, const int* prev_flag, const unsigned long long* prev_parity,
                double factor, unsigned long long floor_ns, unsigned long long cap_ns, cudaStream_t st) {
  arm_kernel<<<1, 1, 0, st>>>(state, prev_flag, prev_parity, factor, floor_ns, cap_ns);
}

void launch_delay(unsigned long long ns, cudaStream_t st) { delay_kernel<<<1, 1, 0, st>>>(ns); }

void launch_to_bf16(const float* in, __nv_bfloat16* out, int64_t n, cudaStream_t st) {
  to_bf16_kernel<<<grid_for(n, 256), 256, 0, st>>>(in, out, n);
}

void launch_transpose_bf16(const __nv_bfloat16* in, __nv_bfloat16* out, int64_t batch, int64_t rows, int64_t cols,
                           cudaStream_t st) {
  dim3 grid((unsigned)((cols + 31) / 32), (unsigned)((rows + 31) / 32), (unsigned)batch);
  transpose_kernel<<<grid, dim3(32, 8), 0, st>>>(in, out, rows, cols);
}

}  // namespace lsb
