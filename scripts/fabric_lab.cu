// L2 -> SM fabric lab: per-launch time of kernels that only stream TMA boxes
// into shared memory (load phase of a tcgen05 GEMM CTA) or only TMA-add-reduce
// fp32 boxes into L2 (split-K epilogue), in CUDA graphs of back-to-back PDL
// launches.  Separates how the BERT-FFN launch time splits between operand
// traffic, reduction traffic and the launch floor.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 scripts/fabric_lab.cu -o /tmp/fabric_lab -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <algorithm>
#include <vector>

#include "../paper_2205_13603_b200/csrc/tc_common.cuh"

using namespace lsb::tc;

#define CK(x)                                                                              \
  do {                                                                                     \
    cudaError_t e_ = (x);                                                                  \
    if (e_ != cudaSuccess) {                                                               \
      fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
      exit(1);                                                                             \
    }                                                                                      \
  } while (0)

struct P {
  int nld;      // 16 KB boxes loaded per CTA
  int shared;   // of which the first `shared` are the same for every CTA (an A operand)
  int nred;     // 16 KB fp32 boxes add-reduced per CTA
  int share;    // CTAs adding into the same C region (split-K ways)
  int how;      // 0 TMA tensor add-reduce, 1 TMA tensor store, 2 red.global.add.v4.f32,
                // 3 st.global.v4, 4 bulk (1-D) add-reduce, 5 TMA add-reduce without the write wait,
                // 6 DSMEM reduce-scatter inside a cluster of `share` CTAs (bulk copies of 16 KB / share
                //   per peer per box), then each CTA TMA-add-reduces its 1/share slice
  float* c;     // the fp32 region buffer (generic-proxy variants)
};

__global__ void __launch_bounds__(128, 1) fabric(const __grid_constant__ CUtensorMap tl,
                                                 const __grid_constant__ CUtensorMap tr, P p) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  __shared__ alignas(8) uint64_t bar, rbar;
  const uint32_t b = smem_u32(&bar), rb = smem_u32(&rbar);
  const uint32_t recv = base + 4 * 16384;  // receive area after the staged boxes
  if (threadIdx.x == 0) {
    mbar_init(b, 1);
    mbar_init(rb, 1);
    if (p.how == 6) mbar_expect_tx(rb, static_cast<uint32_t>(p.nred * (p.share - 1) * (16384 / p.share)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (p.how == 6) cluster_sync_all();
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (threadIdx.x == 0 && p.nld > 0) {
    mbar_expect_tx(b, static_cast<uint32_t>(p.nld) * 16384u);
    for (int i = 0; i < p.nld; ++i) {
      const int row = i < p.shared ? i * 128 : (p.shared + (blockIdx.x * (p.nld - p.shared)) + (i - p.shared)) * 128;
      tma_load_3d(base + i * 16384, &tl, b, 0, row, 0);
    }
  }
  if (p.nld > 0) mbar_wait(b, 0);
  if (p.nred > 0) {
    // smem already holds bytes (whatever was loaded / garbage): reduce them
    fence_proxy_async_smem();
    __syncthreads();
    const int region = blockIdx.x / p.share;
    if (p.how == 0 || p.how == 1 || p.how == 5) {
      if (threadIdx.x == 0) {
        for (int i = 0; i < p.nred; ++i) {
          if (p.how == 1) tma_store_3d(&tr, base + i * 16384, 0, (region * p.nred + i) * 128, 0);
          else tma_reduce_add_3d(&tr, base + i * 16384, 0, (region * p.nred + i) * 128, 0);
        }
        bulk_commit();
        if (p.how == 5) bulk_wait_read();
        else bulk_wait_all();
      }
    } else if (p.how == 6) {
      const uint32_t me = cluster_rank();
      const uint32_t slice = 16384u / static_cast<uint32_t>(p.share);
      if (threadIdx.x == 0) {
        for (int i = 0; i < p.nred; ++i)
          for (int o = 0; o < p.share; ++o) {
            if (o == static_cast<int>(me)) continue;
            const uint32_t src = base + i * 16384 + o * slice;
            const uint32_t dst = map_peer(recv + (i * p.share + me) * slice, o);
            bulk_push_peer(dst, src, slice, map_peer(rb, o));
          }
      }
      mbar_wait(rb, 0);
      // (the sum of the received slices into my slice is ALU work, omitted)
      if (threadIdx.x == 0) {
        const int region = blockIdx.x / p.share;
        for (int i = 0; i < p.nred; ++i)
          tma_reduce_add_3d(&tr, base + i * 16384 + me * slice, 0, (region * p.nred + i) * 128 + me * (128 / p.share), 0);
        bulk_commit();
        bulk_wait_all();
      }
      cluster_sync_all();  // no peer may still push into me when I exit
    } else if (p.how == 4) {
      if (threadIdx.x == 0) {
        for (int i = 0; i < p.nred; ++i) {
          float* dst = p.c + static_cast<int64_t>(region * p.nred + i) * 4096;
          asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], 16384;" ::"l"(dst),
                       "r"(base + i * 16384)
                       : "memory");
        }
        bulk_commit();
        bulk_wait_all();
      }
    } else {
      const float4* src = reinterpret_cast<const float4*>(smem_raw + (base - raw));
      for (int i = 0; i < p.nred; ++i) {
        float4* dst = reinterpret_cast<float4*>(p.c + static_cast<int64_t>(region * p.nred + i) * 4096);
        for (int e = threadIdx.x; e < 1024; e += 128) {
          const float4 v = src[i * 1024 + e];
          if (p.how == 2) red_add_f4(reinterpret_cast<float*>(dst + e), v);
          else dst[e] = v;
        }
      }
    }
  }
  __syncthreads();
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static CUtensorMap map2(void* base, CUtensorMapDataType dt, int esz, int64_t cols, int64_t rows, int bc, int br) {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* q = nullptr;
    cudaDriverEntryPointQueryResult r;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &q, cudaEnableDefault, &r));
    fn = reinterpret_cast<EncodeTiledFn>(q);
  }
  CUtensorMap m;
  cuuint64_t dims[3] = {(cuuint64_t)cols, (cuuint64_t)rows, 1};
  cuuint64_t str[2] = {(cuuint64_t)(cols * esz), (cuuint64_t)(cols * rows * esz)};
  cuuint32_t box[3] = {(cuuint32_t)bc, (cuuint32_t)br, 1};
  cuuint32_t es[3] = {1, 1, 1};
  if (fn(&m, dt, 3, base, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
    fprintf(stderr, "encode failed\n");
    exit(1);
  }
  return m;
}

int main() {
  const int64_t ROWS = 128LL * 2048;  // 2048 distinct 16 KB bf16 boxes (32 MB)
  void *dl, *dr;
  CK(cudaMalloc(&dl, ROWS * 64 * 2));
  CK(cudaMalloc(&dr, ROWS * 32 * 4));
  CK(cudaMemset(dl, 0, ROWS * 64 * 2));
  CK(cudaMemset(dr, 0, ROWS * 32 * 4));
  CUtensorMap tl = map2(dl, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, 64, ROWS, 64, 128);
  CUtensorMap tr = map2(dr, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, 32, ROWS, 32, 128);
  int optin = 0;
  CK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, 0));
  CK(cudaFuncSetAttribute(fabric, cudaFuncAttributeMaxDynamicSharedMemorySize, optin - 1024));
  cudaStream_t st;
  CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  struct C {
    int grid;
    P p;
  };
  std::vector<C> cs;
  for (int g : {144, 288})
    for (int nld : {0, 2, 4, 6, 8}) {
      if (g == 288 && nld > 6) continue;
      cs.push_back({g, {nld, 0, 0, 1, 0, nullptr}});
      if (nld >= 4) cs.push_back({g, {nld, nld / 2, 0, 1, 0, nullptr}});
      if (nld >= 2) cs.push_back({g, {nld, nld, 0, 1, 0, nullptr}});
    }
  for (int g : {144, 288})
    for (int nred : {1, 2})
      for (int how : {0, 1, 6})
        for (int share : {1, 2, 4}) {
          if (how == 6 && share == 1) continue;
          if (how != 6 && share != 1) continue;
          cs.push_back({g, {0, 0, nred, share, how, reinterpret_cast<float*>(dr)}});
        }
  // BERT-FFN shapes: BN 32 / S 12 (288 CTAs: 4 k-tiles of A 16K (shared by 24 N-tiles) + B 4K)
  const int G = 64, R = 7;
  std::vector<std::vector<float>> t(cs.size());
  std::vector<cudaGraphExec_t> ge(cs.size());
  for (size_t i = 0; i < cs.size(); ++i) {
    const int nbox = std::max(std::max(cs[i].p.nld, cs[i].p.nred), 1);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cs[i].grid);
    cfg.blockDim = dim3(128);
    cfg.dynamicSmemBytes = 1024 + 4 * 16384 + nbox * 16384;
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    at[1].id = cudaLaunchAttributeClusterDimension;
    at[1].val.clusterDim.x = cs[i].p.how == 6 ? cs[i].p.share : 1;
    at[1].val.clusterDim.y = 1;
    at[1].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = cs[i].p.how == 6 ? 2 : 1;
    cudaGraph_t g;
    CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    for (int k = 0; k < G; ++k) CK(cudaLaunchKernelEx(&cfg, fabric, tl, tr, cs[i].p));
    CK(cudaStreamEndCapture(st, &g));
    CK(cudaGraphInstantiate(&ge[i], g, 0));
    CK(cudaGraphLaunch(ge[i], st));
  }
  CK(cudaStreamSynchronize(st));
  for (int r = 0; r < R; ++r)
    for (size_t i = 0; i < cs.size(); ++i) {
      CK(cudaGraphLaunch(ge[i], st));
      CK(cudaEventRecord(e0, st));
      CK(cudaGraphLaunch(ge[i], st));
      CK(cudaEventRecord(e1, st));
      CK(cudaEventSynchronize(e1));
      float ms;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      t[i].push_back(ms * 1000.f / G);
    }
  printf("grid nld shared nred share how | median_us  loadMB redMB\n");
  for (size_t i = 0; i < cs.size(); ++i) {
    std::sort(t[i].begin(), t[i].end());
    const P& p = cs[i].p;
    printf("%4d %2d %2d %2d %2d %d | %6.3f  %6.2f %6.2f\n", cs[i].grid, p.nld, p.shared, p.nred, p.share, p.how, t[i][R / 2],
           cs[i].grid * p.nld * 16384 / 1e6, cs[i].grid * p.nred * 16384 / 1e6);
  }
  return 0;
}
