// Launch-floor lab: per-launch time of near-empty kernels in CUDA graphs of
// back-to-back launches, as a function of grid size, dynamic shared memory,
// PDL (programmatic dependent launch) and TMEM allocation -- the fixed cost
// under every tcgen05 candidate launch.  Each configuration is measured in
// several interleaved rounds in one process; the median is reported.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 scripts/launch_lab.cu -o /tmp/launch_lab
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <algorithm>
#include <vector>

#define CK(x)                                                                                  \
  do {                                                                                         \
    cudaError_t e_ = (x);                                                                      \
    if (e_ != cudaSuccess) {                                                                   \
      fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_));     \
      exit(1);                                                                                 \
    }                                                                                          \
  } while (0)

// flags: 1 griddepcontrol (trigger at entry + wait), 2 TMEM alloc/dealloc,
// 4 touch the dynamic smem (one store per thread), 8 trigger after the TMEM alloc
struct Big {
  uint8_t b[640];
};
__global__ void __launch_bounds__(256, 1) probe(int flags, int* sink, const __grid_constant__ Big big) {
  extern __shared__ uint8_t sm[];
  __shared__ uint32_t slot;
  if ((flags & 1) && !(flags & 8)) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (flags & 2) {
    if (threadIdx.x < 32) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(
                       static_cast<uint32_t>(__cvta_generic_to_shared(&slot)))
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  }
  if ((flags & 1) && (flags & 8)) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (flags & 1) asm volatile("griddepcontrol.wait;" ::: "memory");
  if (flags & 4) sm[threadIdx.x * 4] = static_cast<uint8_t>(threadIdx.x);
  if (threadIdx.x == 0 && blockIdx.x == 0 && flags < 0) *sink = sm[0] + big.b[threadIdx.x];
  if (flags & 2) {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (threadIdx.x < 32)
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(slot) : "memory");
  }
}

struct Cfg {
  int grid, threads, smem_kb, flags, pdl, cluster = 0;
};

int main() {
  int optin = 0;
  CK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, 0));
  CK(cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, optin - 1024));
  int* sink;
  CK(cudaMalloc(&sink, 4));
  cudaStream_t st;
  CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  std::vector<Cfg> cs = {
      {144, 128, 0, 0, 0},    {144, 128, 0, 1, 1},    {144, 128, 0, 3, 1},    {144, 128, 0, 11, 1},
      {144, 128, 100, 1, 1},  {144, 128, 100, 3, 1},  {144, 128, 161, 1, 1},  {144, 128, 161, 3, 1},
      {144, 128, 161, 0, 0},  {144, 128, 161, 11, 1}, {288, 128, 81, 1, 1},   {288, 128, 81, 3, 1},
      {288, 128, 81, 0, 0},   {288, 128, 0, 1, 1},    {288, 128, 0, 3, 1},    {148, 128, 161, 3, 1},
      {144, 256, 161, 3, 1},  {72, 128, 161, 3, 1},   {576, 128, 40, 3, 1},   {144, 128, 161, 7, 1},
      {144, 128, 161, 3, 1, 1}, {288, 128, 81, 3, 1, 1}, {144, 128, 161, 3, 1, 2}, {144, 128, 0, 1, 1, 1},
  };
  const int G = 64, R = 7;
  std::vector<std::vector<float>> t(cs.size());
  std::vector<cudaGraphExec_t> ge(cs.size());
  for (size_t i = 0; i < cs.size(); ++i) {
    const Cfg& c = cs[i];
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(c.grid);
    cfg.blockDim = dim3(c.threads);
    cfg.dynamicSmemBytes = static_cast<size_t>(c.smem_kb) * 1024;
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = c.pdl;
    at[1].id = cudaLaunchAttributeClusterDimension;
    at[1].val.clusterDim.x = c.cluster ? c.cluster : 1;
    at[1].val.clusterDim.y = 1;
    at[1].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = c.cluster ? 2 : 1;
    cudaGraph_t g;
    CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    Big big{};
    for (int k = 0; k < G; ++k) CK(cudaLaunchKernelEx(&cfg, probe, c.flags, sink, big));
    CK(cudaStreamEndCapture(st, &g));
    CK(cudaGraphInstantiate(&ge[i], g, 0));
    CK(cudaGraphLaunch(ge[i], st));
  }
  CK(cudaStreamSynchronize(st));
  for (int r = 0; r < R; ++r)
    for (size_t i = 0; i < cs.size(); ++i) {
      CK(cudaGraphLaunch(ge[i], st));  // warm
      CK(cudaEventRecord(e0, st));
      CK(cudaGraphLaunch(ge[i], st));
      CK(cudaEventRecord(e1, st));
      CK(cudaEventSynchronize(e1));
      float ms;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      t[i].push_back(ms * 1000.f / G);
    }
  printf("grid threads smemKB flags pdl cluster | median_us min_us   (640-byte __grid_constant__ param)\n");
  for (size_t i = 0; i < cs.size(); ++i) {
    std::sort(t[i].begin(), t[i].end());
    printf("%4d %4d %4d %3d %d %d | %6.3f %6.3f\n", cs[i].grid, cs[i].threads, cs[i].smem_kb, cs[i].flags, cs[i].pdl,
           cs[i].cluster,
           t[i][R / 2], t[i][0]);
  }
  return 0;
}
