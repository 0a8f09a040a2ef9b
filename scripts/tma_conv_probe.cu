// TMA throughput of the conv kernel's operand pattern: per CTA, K boxes of
// {64 ch, 8 w, 8 h, 1 n} bf16 (4-D map over a 1x56x56x64 NHWC tensor, taps
// shifted by -1..1 with OOB fill) vs the same bytes as 2-D {64, 64} boxes.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 tma_conv_probe.cu -lcuda -o tma_conv_probe
#include <cstdio>
#include <cuda.h>
#include <cuda_runtime.h>
#include <vector>
#include <algorithm>

__device__ __forceinline__ unsigned long long gt() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void probe(const __grid_constant__ CUtensorMap m4, const __grid_constant__ CUtensorMap m2, int mode,
                      int nbox, int all_at_once, unsigned long long* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ unsigned long long bar[16];
  uint32_t dst = ((uint32_t)__cvta_generic_to_shared(sm) + 1023) & ~1023u;
  if (threadIdx.x == 0) {
    for (int i = 0; i < nbox; ++i)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&bar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&m4));
    asm volatile("prefetch.tensormap [%0];" ::"l"(&m2));
    const int box = blockIdx.x;  // 7x7 pixel boxes
    const int bh = (box / 7) * 8, bw = (box % 7) * 8;
    unsigned long long t0 = gt(), tf = 0;
    for (int i = 0; i < nbox; ++i) {
      uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar[i]);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(8192));
      if (mode == 0) {
        const int r = i / 3 - 1, s = i % 3 - 1;
        asm volatile(
            "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
            ::"r"(dst + i * 8192), "l"(&m4), "r"(0), "r"(bw + s), "r"(bh + r), "r"(0), "r"(b) : "memory");
      } else {
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
            ::"r"(dst + i * 8192), "l"(&m2), "r"(0), "r"((box * 9 + i) % 49 * 64), "r"(b) : "memory");
      }
      if (!all_at_once) {
        uint32_t ok = 0;
        while (!ok)
          asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0,1,0,p;}"
                       : "=r"(ok) : "r"(b) : "memory");
      }
    }
    for (int i = 0; i < nbox; ++i) {
      uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar[i]);
      uint32_t ok = 0;
      while (!ok)
        asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0,1,0,p;}"
                     : "=r"(ok) : "r"(b) : "memory");
      if (i == 0) tf = gt();
    }
    unsigned long long t1 = gt();
    out[blockIdx.x * 2] = tf - t0;
    out[blockIdx.x * 2 + 1] = t1 - t0;
  }
}

typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  void* X;
  cudaMalloc(&X, 56 * 56 * 64 * 2 * 2);
  cudaMemset(X, 0, 56 * 56 * 64 * 2 * 2);
  EncFn enc;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  CUtensorMap m4, m2;
  cuuint64_t d4[4] = {64, 56, 56, 1}, s4[3] = {128, 56 * 128, 56 * 56 * 128};
  cuuint32_t b4[4] = {64, 8, 8, 1}, e4[4] = {1, 1, 1, 1};
  enc(&m4, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, X, d4, s4, b4, e4, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  cuuint64_t d2[2] = {64, 56 * 56}, s2[1] = {128};
  cuuint32_t b2[2] = {64, 64}, e2[2] = {1, 1};
  enc(&m2, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, X, d2, s2, b2, e2, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  unsigned long long* out;
  cudaMalloc(&out, 49 * 2 * 8);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int mode = 0; mode < 2; ++mode)
    for (int all = 0; all < 2; ++all)
      for (int rep = 0; rep < 3; ++rep) {
        probe<<<49, 128, 9 * 8192 + 1024>>>(m4, m2, mode, 9, all, out);
        cudaDeviceSynchronize();
        std::vector<unsigned long long> h(98);
        cudaMemcpy(h.data(), out, 98 * 8, cudaMemcpyDeviceToHost);
        std::vector<double> f, t;
        for (int i = 0; i < 49; ++i) { f.push_back(h[2 * i]); t.push_back(h[2 * i + 1]); }
        std::sort(f.begin(), f.end()); std::sort(t.begin(), t.end());
        printf("%s %s rep %d: first box med %.0f ns, all 9 boxes med %.0f max %.0f ns\n", mode ? "2-D" : "4-D",
               all ? "all-at-once" : "serial", rep, f[24], t[24], t[48]);
      }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
