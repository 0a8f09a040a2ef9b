// GEMM lab 3: the bmm QK^T launch (12 x [128x64] x [64x128] -> fp32, one
// 64-deep k-tile per CTA) -- where its ~2.8 us go and which epilogue is
// shortest.  Per CTA: one TMA stage (A 128x64, B BNx64), 4 UMMAs into TMEM,
// then one of
//   E0 TMEM -> padded smem -> coalesced float4 stores (the product's BN%32!=0 path)
//   E1 TMEM -> registers -> st.global.v4 of each thread's own row (no smem)
//   E2 TMEM -> swizzled smem -> TMA store, wait for the smem reads only
//   E3 as E2, wait for the bulk group to complete
// Exactness on small-integer inputs; per-launch time from CUDA graphs of 64
// PDL launches, median of 7 interleaved rounds.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Ipaper_2205_13603_b200/csrc scripts/gemm_lab3.cu -o /tmp/gemm_lab3 -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <vector>

#include "../paper_2205_13603_b200/csrc/tc_common.cuh"
// the product kernel, launched through its own launcher (variant "product")
#include "../paper_2205_13603_b200/csrc/tc_gemm.cu"
namespace lsb {
int opt_in_dynamic_smem(const void* fn) {
  int dev = 0, optin = 0;
  cudaFuncAttributes fa;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  cudaFuncGetAttributes(&fa, fn);
  const int dyn = optin - static_cast<int>(fa.sharedSizeBytes);
  return cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn) == cudaSuccess ? dyn : 0;
}
}  // namespace lsb

using namespace lsb::tc;

#define CK(x)                                                                              \
  do {                                                                                     \
    cudaError_t e_ = (x);                                                                  \
    if (e_ != cudaSuccess) {                                                               \
      fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
      exit(1);                                                                             \
    }                                                                                      \
  } while (0)

constexpr int B = 12, M = 128, N = 128, K = 64;

struct P {
  unsigned long long* tr;  // optional per-CTA stamps, the product kernel's slots (0 start, 1 setup,
                           // 2 operands landed, 3 accumulator done, 6 stored)
  int BN, epi, ld;
  int trig;  // where griddepcontrol.launch_dependents is issued: 0 before the wait, 1 after it, 2 after the MMAs
  float* c;
  uint32_t idesc, cols;
};

__global__ void __launch_bounds__(128, 1)
lab3(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb,
     const __grid_constant__ CUtensorMap tc, P p) {
  extern __shared__ uint8_t smem_raw[];
  __shared__ uint32_t s_slot;
  __shared__ __align__(8) uint64_t s_bar[2];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* gbase = smem_raw + (base - raw);
  const uint32_t sa = base, sb = base + M * 128;
  const uint32_t full = smem_u32(&s_bar[0]), done = smem_u32(&s_bar[1]);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nb = blockIdx.x, batch = blockIdx.y;
  unsigned long long* tr = p.tr ? p.tr + 8 * (blockIdx.y * gridDim.x + blockIdx.x) : nullptr;
  if (tr && threadIdx.x == 0) tr[0] = gtime();
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&s_slot)),
                 "r"(p.cols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (threadIdx.x == 32) {
    mbar_init(full, 1);
    mbar_init(done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&ta)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tb)) : "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = s_slot;
  if (tr && threadIdx.x == 0) tr[1] = gtime();
  if (p.trig == 0) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (p.trig == 1) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (threadIdx.x == 0) {
    mbar_expect_tx(full, M * 128 + p.BN * 128);
    tma_load_3d(sa, &ta, full, 0, 0, batch);
    tma_load_3d(sb, &tb, full, 0, nb * p.BN, batch);
  } else if (threadIdx.x == 32) {
    mbar_wait(full, 0);
    tc_fence_after();
    if (tr) tr[2] = gtime();
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) umma_bf16(tmem, sdesc(sa + kk * 32), sdesc(sb + kk * 32), p.idesc, kk != 0);
    umma_commit(done);
  }
  mbar_wait(done, 0);
  if (tr && threadIdx.x == 0) tr[3] = gtime();
  if (p.trig == 2) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  __syncwarp();
  tc_fence_after();
  const int row = warp * 32 + lane;
  const uint32_t trow = tmem + (static_cast<uint32_t>(warp * 32) << 16);
  float* ctile = p.c + static_cast<int64_t>(batch) * M * N + nb * p.BN;
  if (p.epi == 1) {
    float* dst = ctile + static_cast<int64_t>(row) * N;
    for (int c0 = 0; c0 < p.BN; c0 += 16) {
      uint32_t v[16];
      tmem_ld16_nowait(trow + c0, v);
      tmem_wait();
#pragma unroll
      for (int q = 0; q < 4; ++q)
        *reinterpret_cast<float4*>(dst + c0 + 4 * q) =
            make_float4(__uint_as_float(v[4 * q]), __uint_as_float(v[4 * q + 1]), __uint_as_float(v[4 * q + 2]),
                        __uint_as_float(v[4 * q + 3]));
    }
  } else if (p.epi == 0) {
    float* stg = reinterpret_cast<float*>(gbase) + row * p.ld;  // over the finished operand stage
    for (int c0 = 0; c0 < p.BN; c0 += 16) {
      uint32_t v[16];
      tmem_ld16_nowait(trow + c0, v);
      tmem_wait();
#pragma unroll
      for (int q = 0; q < 4; ++q)
        *reinterpret_cast<float4*>(stg + c0 + 4 * q) =
            make_float4(__uint_as_float(v[4 * q]), __uint_as_float(v[4 * q + 1]), __uint_as_float(v[4 * q + 2]),
                        __uint_as_float(v[4 * q + 3]));
    }
    __syncthreads();
    const int c4 = p.BN / 4;
    const float* st = reinterpret_cast<const float*>(gbase);
    for (int e = threadIdx.x; e < 128 * c4; e += 128) {
      const int r = e / c4, cc = (e % c4) * 4;
      *reinterpret_cast<float4*>(ctile + static_cast<int64_t>(r) * N + cc) =
          *reinterpret_cast<const float4*>(st + r * p.ld + cc);
    }
  } else {
    for (int c0 = 0; c0 < p.BN; c0 += 32) {
      uint32_t v[32];
      tmem_ld16_nowait(trow + c0, v);
      tmem_ld16_nowait(trow + c0 + 16, v + 16);
      tmem_wait();
      uint8_t* chunk = gbase + (c0 / 32) * 16384 + row * 128;
#pragma unroll
      for (int q = 0; q < 8; ++q)
        *reinterpret_cast<float4*>(chunk + ((q ^ (row & 7)) << 4)) =
            make_float4(__uint_as_float(v[4 * q]), __uint_as_float(v[4 * q + 1]), __uint_as_float(v[4 * q + 2]),
                        __uint_as_float(v[4 * q + 3]));
    }
    fence_proxy_async_smem();
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int c0 = 0; c0 < p.BN; c0 += 32) tma_store_3d(&tc, base + (c0 / 32) * 16384, nb * p.BN + c0, 0, batch);
      bulk_commit();
      if (p.epi == 2) bulk_wait_read();
      else bulk_wait_all();
    }
  }
  if (tr && threadIdx.x == 0) tr[6] = gtime();
  tc_fence_before();
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(p.cols) : "memory");
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static CUtensorMap map3(void* base, CUtensorMapDataType dt, int esz, int64_t d0, int64_t d1, int64_t d2, int b0,
                        int b1) {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* q = nullptr;
    cudaDriverEntryPointQueryResult r;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &q, cudaEnableDefault, &r));
    fn = reinterpret_cast<EncodeTiledFn>(q);
  }
  CUtensorMap m;
  cuuint64_t dims[3] = {(cuuint64_t)d0, (cuuint64_t)d1, (cuuint64_t)d2};
  cuuint64_t str[2] = {(cuuint64_t)(d0 * esz), (cuuint64_t)(d0 * d1 * esz)};
  cuuint32_t box[3] = {(cuuint32_t)b0, (cuuint32_t)b1, 1};
  cuuint32_t es[3] = {1, 1, 1};
  if (fn(&m, dt, 3, base, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
    fprintf(stderr, "encode failed\n");
    exit(1);
  }
  return m;
}

static uint16_t f2bf(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  return static_cast<uint16_t>(u >> 16);
}

int main() {
  // Q [B][M][K], Kmat [B][N][K] (both K-major), C [B][M][N] fp32
  std::vector<uint16_t> hq(B * M * K), hk(B * N * K);
  std::vector<float> fq(B * M * K), fk(B * N * K);
  uint32_t s = 4242;
  for (size_t i = 0; i < fq.size(); ++i) {
    s = s * 1664525u + 1013904223u;
    fq[i] = static_cast<float>(static_cast<int>((s >> 24) % 7) - 3);
    hq[i] = f2bf(fq[i]);
  }
  for (size_t i = 0; i < fk.size(); ++i) {
    s = s * 1664525u + 1013904223u;
    fk[i] = static_cast<float>(static_cast<int>((s >> 24) % 7) - 3);
    hk[i] = f2bf(fk[i]);
  }
  std::vector<double> ref(B * M * N);
  for (int b = 0; b < B; ++b)
    for (int m = 0; m < M; ++m)
      for (int n = 0; n < N; ++n) {
        double acc = 0;
        for (int k = 0; k < K; ++k) acc += static_cast<double>(fq[(b * M + m) * K + k]) * fk[(b * N + n) * K + k];
        ref[(b * M + m) * N + n] = acc;
      }
  void *dq, *dk;
  float* dc;
  CK(cudaMalloc(&dq, hq.size() * 2));
  CK(cudaMalloc(&dk, hk.size() * 2));
  CK(cudaMalloc(&dc, B * M * N * 4));
  CK(cudaMemcpy(dq, hq.data(), hq.size() * 2, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dk, hk.data(), hk.size() * 2, cudaMemcpyHostToDevice));
  CK(cudaFuncSetAttribute(lab3, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  CUtensorMap tmq = map3(dq, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, K, M, B, 64, 128);
  CUtensorMap tmcm = map3(dc, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, N, M, B, 32, 128);
  cudaStream_t st;
  CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  struct V {
    int BN, epi, G, trig;
  };
  std::vector<V> vs;
  for (int bn : {16, 32, 64, 128})
    for (int epi = 0; epi < 4; ++epi)
      if (epi < 2 || bn % 32 == 0) vs.push_back({bn, epi, 64, 0});
  // graph length (launches per graph, PDL edges between them) x trigger position
  for (int g : {64, 2000}) {
    vs.push_back({16, 4, g, 1});
    vs.push_back({32, 4, g, 1});
    vs.push_back({64, 4, g, 1});
  }
  for (int trig = 0; trig < 3; ++trig)
    for (int g : {64, 256, 2000}) {
      if (trig == 0 && g == 64) continue;
      vs.push_back({16, 1, g, trig});
      vs.push_back({32, 1, g, trig});
      vs.push_back({64, 2, g, trig});
      vs.push_back({128, 2, g, trig});
    }
  std::vector<cudaGraphExec_t> ge(vs.size());
  std::vector<std::vector<float>> t(vs.size());
  std::vector<int> ok(vs.size());
  for (size_t i = 0; i < vs.size(); ++i) {
    const V& v = vs[i];
    P p{};
    p.BN = v.BN;
    p.epi = v.epi;
    p.ld = v.BN + 4;
    p.trig = v.trig;
    p.c = dc;
    p.idesc = (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(v.BN >> 3) << 17) |
              (static_cast<uint32_t>(128 >> 4) << 24);
    p.cols = 32;
    while (p.cols < static_cast<uint32_t>(v.BN)) p.cols <<= 1;
    const int stage = M * 128 + v.BN * 128;
    const int epi_bytes = v.epi >= 2 ? (v.BN / 32) * 16384 : 128 * (v.BN + 4) * 4;
    const int smem = 1024 + std::max(stage, epi_bytes);
    CUtensorMap tmk = map3(dk, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, K, N, B, 64, v.BN);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(N / v.BN, B);
    cfg.blockDim = dim3(128);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    CK(cudaStreamSynchronize(st));
    CK(cudaMemset(dc, 0xff, B * M * N * 4));
    CK(cudaDeviceSynchronize());
    lsb::TcLaunch L;
    L.tmap_a = &tmq;
    L.tmap_b = &tmk;
    L.tmap_c = &tmcm;
    L.c = dc;
    L.sc_b = M * N;
    L.sc_m = N;
    L.m = M;
    L.n = N;
    L.k = K;
    L.bn = v.BN;
    L.splits = 1;
    L.kt = 1;
    L.stages = 1;
    L.batch = B;
    L.grid_m = 1;
    L.grid_n = N / v.BN;
    L.smem_bytes = static_cast<int>(lsb::tc_geom(v.BN, 1, 1, B * (N / v.BN)).smem);
    auto launch = [&]() {
      if (v.epi == 4) {
        if (!lsb::launch_tc_gemm(L, st)) {
          fprintf(stderr, "product launch failed\n");
          exit(1);
        }
      } else {
        CK(cudaLaunchKernelEx(&cfg, lab3, tmq, tmk, tmcm, p));
      }
    };
    launch();
    CK(cudaStreamSynchronize(st));
    std::vector<float> hc(B * M * N);
    CK(cudaMemcpy(hc.data(), dc, hc.size() * 4, cudaMemcpyDeviceToHost));
    bool exact = true;
    for (size_t k = 0; k < hc.size() && exact; ++k) exact = static_cast<double>(hc[k]) == ref[k];
    ok[i] = exact;
    cudaGraph_t g;
    CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    for (int k = 0; k < v.G; ++k) launch();
    CK(cudaStreamEndCapture(st, &g));
    CK(cudaGraphInstantiate(&ge[i], g, 0));
    CK(cudaGraphLaunch(ge[i], st));
  }
  CK(cudaStreamSynchronize(st));
  for (int r = 0; r < 7; ++r)
    for (size_t i = 0; i < vs.size(); ++i) {
      CK(cudaGraphLaunch(ge[i], st));
      CK(cudaEventRecord(e0, st));
      CK(cudaGraphLaunch(ge[i], st));
      CK(cudaEventRecord(e1, st));
      CK(cudaEventSynchronize(e1));
      float ms;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      t[i].push_back(ms * 1000.f / vs[i].G);
    }
  const char* names[5] = {"staged+coalesced", "register st.global", "TMA store, wait read", "TMA store, wait all",
                          "product tc_gemm_kernel"};
  const char* trigs[3] = {"trigger before wait", "trigger after wait", "trigger after MMA"};
  printf("BN ctas epilogue              G  trigger             | median_us min_us exact\n");
  for (size_t i = 0; i < vs.size(); ++i) {
    std::sort(t[i].begin(), t[i].end());
    printf("%3d %3d %-22s %4d %-19s | %5.2f %5.2f %s\n", vs[i].BN, (N / vs[i].BN) * B, names[vs[i].epi], vs[i].G,
           trigs[vs[i].trig], t[i][3], t[i][0],
           ok[i] ? "exact" : "MISMATCH");
  }
  // timelines: one traced graph of 64 launches per kernel (BN 16, register
  // epilogue vs the product kernel), medians over launches 8..63
  {
    const int TG = 64, ctas = 96;
    unsigned long long* dtr;
    CK(cudaMalloc(&dtr, sizeof(unsigned long long) * 8 * ctas * TG));
    for (int which = 0; which < 2; ++which) {
      CK(cudaMemset(dtr, 0, sizeof(unsigned long long) * 8 * ctas * TG));
      P p{};
      p.BN = 16;
      p.epi = 1;
      p.ld = 20;
      p.trig = 1;
      p.c = dc;
      p.idesc = (1u << 4) | (1u << 7) | (1u << 10) | (2u << 17) | (8u << 24);
      p.cols = 32;
      CUtensorMap tmk = map3(dk, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, K, N, B, 64, 16);
      lsb::TcLaunch L;
      L.tmap_a = &tmq;
      L.tmap_b = &tmk;
      L.tmap_c = &tmcm;
      L.c = dc;
      L.sc_b = M * N;
      L.sc_m = N;
      L.m = M;
      L.n = N;
      L.k = K;
      L.bn = 16;
      L.splits = 1;
      L.kt = 1;
      L.stages = 1;
      L.batch = B;
      L.grid_m = 1;
      L.grid_n = 8;
      L.smem_bytes = static_cast<int>(lsb::tc_geom(16, 1, 1, 96).smem);
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(8, B);
      cfg.blockDim = dim3(128);
      cfg.dynamicSmemBytes = 1024 + 18432;
      cfg.stream = st;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      cudaGraph_t g;
      cudaGraphExec_t gx;
      CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
      for (int k = 0; k < TG; ++k) {
        unsigned long long* t0 = dtr + static_cast<size_t>(k) * 8 * ctas;
        if (which) {
          L.trace = t0;
          lsb::launch_tc_gemm(L, st);
        } else {
          p.tr = t0;
          CK(cudaLaunchKernelEx(&cfg, lab3, tmq, tmk, tmcm, p));
        }
      }
      CK(cudaStreamEndCapture(st, &g));
      CK(cudaGraphInstantiate(&gx, g, 0));
      CK(cudaGraphLaunch(gx, st));
      CK(cudaGraphLaunch(gx, st));
      CK(cudaStreamSynchronize(st));
      std::vector<unsigned long long> h(static_cast<size_t>(8) * ctas * TG);
      CK(cudaMemcpy(h.data(), dtr, h.size() * 8, cudaMemcpyDeviceToHost));
      std::vector<double> per, gap, land, mma, epi, setup;
      for (int k = 8; k < TG; ++k) {
        const unsigned long long* a = h.data() + static_cast<size_t>(k) * 8 * ctas;
        unsigned long long e_max = 0, l_min = ~0ull;
        for (int c = 0; c < ctas; ++c) {
          e_max = std::max(e_max, a[8 * c + 6]);
          l_min = std::min(l_min, a[8 * c + 2]);
          setup.push_back(static_cast<double>(a[8 * c + 1] - a[8 * c + 0]));
          mma.push_back(static_cast<double>(a[8 * c + 3] - a[8 * c + 2]));
          epi.push_back(static_cast<double>(a[8 * c + 6] - a[8 * c + 3]));
        }
        if (k + 1 < TG) {
          const unsigned long long* b = a + 8 * ctas;
          unsigned long long e2 = 0, l2 = ~0ull;
          for (int c = 0; c < ctas; ++c) {
            e2 = std::max(e2, b[8 * c + 6]);
            l2 = std::min(l2, b[8 * c + 2]);
          }
          per.push_back(static_cast<double>(e2 - e_max));
          gap.push_back(static_cast<double>(l2 - e_max));
          land.push_back(static_cast<double>(e2 - l2));
        }
      }
      auto med = [](std::vector<double> v) {
        std::sort(v.begin(), v.end());
        return v.empty() ? 0.0 : v[v.size() / 2];
      };
      printf("timeline %-8s: end-to-end per launch %6.0f ns | last end -> next first operands landed %6.0f ns | "
             "first landed -> last end %6.0f ns | per CTA: setup %4.0f, landed->acc %4.0f, acc->stored %4.0f ns\n",
             which ? "product" : "lab E1", med(per), med(gap), med(land), med(setup), med(mma), med(epi));
    }
  }
  return 0;
}
