// Launch floor on B200: back-to-back launches of an empty kernel captured in
// a CUDA graph, with/without PDL and with thread-block clusters.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 launch_floor.cu -o launch_floor
#include <cstdio>
#include <cuda_runtime.h>

__global__ void empty_kernel(int* p) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (p && threadIdx.x == 0 && blockIdx.x == 100000) p[0] = 1;
}

static float run(int grid, int cluster, bool pdl, int reps) {
  cudaStream_t st;
  cudaStreamCreate(&st);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(128);
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cluster; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = pdl;
  cfg.attrs = at; cfg.numAttrs = 2;
  if (cluster > 8) cudaFuncSetAttribute(empty_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaGraph_t g; cudaGraphExec_t ge;
  cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
  for (int i = 0; i < reps; ++i) cudaLaunchKernelEx(&cfg, empty_kernel, (int*)nullptr);
  cudaStreamEndCapture(st, &g);
  cudaGraphInstantiate(&ge, g, 0);
  cudaGraphLaunch(ge, st);
  cudaStreamSynchronize(st);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a, st);
  cudaGraphLaunch(ge, st);
  cudaEventRecord(b, st);
  cudaStreamSynchronize(st);
  float ms; cudaEventElapsedTime(&ms, a, b);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("err %s\n", cudaGetErrorString(e));
  return ms * 1e3f / reps;
}

int main() {
  int grids[] = {1, 96, 144, 148, 192, 296};
  int clusters[] = {1, 2, 4, 8, 16};
  for (int pdl = 0; pdl < 2; ++pdl)
    for (int c : clusters)
      for (int g : grids) {
        if (g % c) continue;
        float r3 = run(g, c, pdl, 3), r100 = run(g, c, pdl, 100);
        printf("pdl %d cluster %2d grid %3d : reps3 %.2f us/launch  reps100 %.2f us/launch\n", pdl, c, g, r3, r100);
      }
  return 0;
}
