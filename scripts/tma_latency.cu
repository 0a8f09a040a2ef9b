// TMA first-load latency probe: one 128x64 bf16 box (16 KB, 128B swizzle)
// per CTA, globaltimer around issue -> mbarrier completion, cold then warm.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 tma_latency.cu -lcuda -o tma_latency
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

__global__ void probe(const __grid_constant__ CUtensorMap map, const CUtensorMap* gmap, int use_gmap, int boxes,
                      unsigned long long* out, const int* g) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ unsigned long long bar;
  uint32_t sbar = (uint32_t)__cvta_generic_to_shared(&bar);
  uint32_t dst = ((uint32_t)__cvta_generic_to_shared(sm) + 1023) & ~1023u;
  const CUtensorMap* m = use_gmap ? gmap : &map;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sbar));
    asm volatile("fence.mbarrier_init.release.cluster;");
    asm volatile("prefetch.tensormap [%0];" ::"l"(m));
    unsigned long long t[4];
    // plain global load latency
    t[0] = gt();
    int v = *(volatile const int*)(g + blockIdx.x * 64);
    t[1] = gt();
    for (int r = 0; r < 2; ++r) {
      unsigned long long a = gt();
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sbar), "r"(boxes * 16384));
      for (int b = 0; b < boxes; ++b)
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
            ::"r"(dst + b * 16384), "l"(m), "r"((int)((blockIdx.x * boxes + b) % 48) * 64), "r"(0), "r"(0), "r"(sbar)
            : "memory");
      uint32_t ok = 0;
      while (!ok)
        asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                     : "=r"(ok) : "r"(sbar), "r"(r & 1) : "memory");
      t[2 + r] = gt() - a;
    }
    out[blockIdx.x * 4 + 0] = t[1] - t[0];
    out[blockIdx.x * 4 + 1] = t[2];
    out[blockIdx.x * 4 + 2] = t[3];
    out[blockIdx.x * 4 + 3] = v;
  }
}

typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  void* A;
  cudaMalloc(&A, 128 * 3072 * 2);
  cudaMemset(A, 0, 128 * 3072 * 2);
  int* g;
  cudaMalloc(&g, 1 << 20);
  cudaMemset(g, 0, 1 << 20);
  EncFn enc;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  CUtensorMap map;
  cuuint64_t dims[3] = {3072, 128, 1};
  cuuint64_t str[2] = {3072 * 2, 128 * 3072 * 2};
  cuuint32_t box[3] = {64, 128, 1}, es[3] = {1, 1, 1};
  enc(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, A, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  CUtensorMap* gmap;
  cudaMalloc(&gmap, sizeof map);
  cudaMemcpy(gmap, &map, sizeof map, cudaMemcpyHostToDevice);
  unsigned long long* out;
  cudaMalloc(&out, 148 * 4 * 8);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  int grids[] = {1, 148};
  int boxes_l[] = {1, 4, 8};
  for (int use_g = 0; use_g < 2; ++use_g)
    for (int grid : grids)
      for (int boxes : boxes_l)
        for (int rep = 0; rep < 2; ++rep) {
          probe<<<grid, 128, boxes * 16384 + 1024>>>(map, gmap, use_g, boxes, out, g);
          cudaDeviceSynchronize();
          std::vector<unsigned long long> h(grid * 4);
          cudaMemcpy(h.data(), out, grid * 4 * 8, cudaMemcpyDeviceToHost);
          std::vector<double> ld, t1, t2;
          for (int i = 0; i < grid; ++i) { ld.push_back(h[i*4]); t1.push_back(h[i*4+1]); t2.push_back(h[i*4+2]); }
          std::sort(ld.begin(), ld.end()); std::sort(t1.begin(), t1.end()); std::sort(t2.begin(), t2.end());
          printf("gmap %d grid %3d boxes %d launch %d: ldg %.0f ns | tma#1 med %.0f max %.0f ns | tma#2 med %.0f max %.0f ns\n",
                 use_g, grid, boxes, rep, ld[grid/2], t1[grid/2], t1[grid-1], t2[grid/2], t2[grid-1]);
        }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
