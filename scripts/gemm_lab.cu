// Standalone tcgen05 GEMM lab for the BERT-FFN shape (M=128, N=768, K=3072):
// times split-K / multicast / reduction variants of one UMMA tile per CTA in
// CUDA graphs of back-to-back PDL launches, and checks C bit-exactly against
// a host reference on small-integer inputs.  Not product code: it decides
// which implementation the runner's tc_gemm family uses.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lcuda scripts/gemm_lab.cu -o gpurun_out/gemm_lab
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <string>
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
  int N, K, BN, S, KT, CN, red, skip, ST;  // ST: ring stages (k-tiles in flight)
  unsigned long long* tr;  // optional per-CTA %globaltimer stamps (9 per CTA)
  float* c;
  float* ws;
  uint32_t* cnt;   // per tile arrival counter (never reset: epochs)
  uint32_t* flag;  // per tile zero-release flag (red 0)
  uint32_t idesc, tmem_cols;
};

constexpr int kA = 128 * 64 * 2;

__global__ void __launch_bounds__(128, 1)
lab_kernel(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb,
           const __grid_constant__ CUtensorMap tc, const __grid_constant__ CUtensorMap tw, P p) {
  extern __shared__ uint8_t smem_raw[];
  __shared__ uint32_t s_ticket;
  __shared__ volatile uint32_t s_ready;
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* gbase = smem_raw + (base - raw);
  const int bbytes = p.BN * 128;
  const uint32_t a0 = base, b0 = base + p.ST * kA;
  const uint32_t ring = p.ST * (kA + bbytes);
  const uint32_t stg = static_cast<uint32_t>(p.BN / 32) * 16384u;
  const uint32_t bars = base + (ring > stg ? ring : stg);
  const uint32_t full = bars, empty = bars + 8 * p.ST, done = bars + 16 * p.ST;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(gbase + (done + 16 - base));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nb = blockIdx.x, split = blockIdx.z;
  const int tile = nb;
  unsigned long long* tr = p.tr ? p.tr + 9 * (blockIdx.z * gridDim.x + blockIdx.x) : nullptr;
  if (tr && threadIdx.x == 0) {
    tr[0] = gtime();
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    tr[8] = smid;
  }

  if (p.skip & 8) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (warp == 0 && !(p.skip & 4)) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tslot)),
                 "r"(p.tmem_cols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (threadIdx.x == 0) s_ready = 0;
  if (threadIdx.x == 32 && !(p.skip & 32)) {
    for (int s = 0; s < p.ST; ++s) {
      mbar_init(full + 8 * s, 1);
      mbar_init(empty + 8 * s, 1);
    }
    mbar_init(done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&ta)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tb)) : "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = (p.skip & 4) ? 0u : *tslot;
  if (p.CN > 1) cluster_arrive();
  if (tr && threadIdx.x == 0) tr[1] = gtime();
  // skip 64: weight (B) k-tiles of the first ring fill issued before the
  // dependency wait (read-only operand); skip 128: the A k-tiles too
  const int pre = (p.skip & 64) && !(p.skip & 1) ? (p.ST < p.KT ? p.ST : p.KT) : 0;
  if (pre && warp == 0 && lane == 0) {
    for (int kt = 0; kt < pre; ++kt) {
      const int kc = (split * p.KT + kt) * 64;
      mbar_expect_tx(full + 8 * kt, kA + bbytes);
      tma_load_3d(b0 + kt * bbytes, &tb, full + 8 * kt, kc, nb * p.BN, 0);
      if (p.skip & 128) tma_load_3d(a0 + kt * kA, &ta, full + 8 * kt, kc, 0, 0);
    }
  }
  asm volatile("griddepcontrol.wait;" ::: "memory");
  // default: trigger the next grid after the wait (as the product kernel;
  // skip 8 triggers at kernel start instead)
  if (!(p.skip & 8)) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (tr && threadIdx.x == 0) tr[2] = gtime();
  if (p.CN > 1) cluster_wait();

  float* ctile = p.c + static_cast<int64_t>(nb) * p.BN;
  const int c4 = p.BN / 4;
  if (p.red == 0 && p.S > 1 && warp >= 2 && !(p.skip & 256)) {
    const int t2 = threadIdx.x - 64;
    if (t2 == 0) s_ticket = atomicAdd(p.cnt + tile, 1u);
    asm volatile("bar.sync 1, 64;" ::: "memory");
    const uint32_t t = s_ticket;
    if (t % static_cast<uint32_t>(p.S) == 0) {
      const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int e = t2; e < 128 * c4; e += 64) {
        const int r = e / c4, cc = (e % c4) * 4;
        *reinterpret_cast<float4*>(ctile + static_cast<int64_t>(r) * p.N + cc) = z;
      }
      asm volatile("bar.sync 1, 64;" ::: "memory");
      if (t2 == 0) st_release_u32(p.flag + tile, t / p.S + 1);
    } else if ((p.skip & 512) && t2 == 0) {
      // skip 512: observe the tile's zeroing while the operands stream in
      while (ld_acquire_u32(p.flag + tile) < t / p.S + 1) __nanosleep(32);
      s_ready = 1;
    }
  }

  if (!(p.skip & 1)) {
    if (warp == 0 && lane == 0) {
      const int rank = p.CN > 1 ? static_cast<int>(cluster_rank()) : 0;
      const int rows = 128 / p.CN;
      const uint16_t mask = static_cast<uint16_t>((1u << p.CN) - 1u);
      for (int kt = 0; kt < p.KT; ++kt) {
        const int kc = (split * p.KT + kt) * 64;
        const int s = kt % p.ST;
        if (kt < pre) {  // B (and A) already in flight
          if (!(p.skip & 128)) tma_load_3d(a0 + s * kA, &ta, full + 8 * s, kc, 0, 0);
          continue;
        }
        if (kt >= p.ST) mbar_wait(empty + 8 * s, ((kt / p.ST) & 1) ^ 1);
        mbar_expect_tx(full + 8 * s, kA + bbytes);
        if (p.CN > 1)  // ta's box is {64, 128 / CN}: my row slice, into every CTA of the cluster
          tma_load_3d_mc(a0 + s * kA + rank * rows * 128, &ta, full + 8 * s, kc, rank * rows, 0, mask);
        else
          tma_load_3d(a0 + s * kA, &ta, full + 8 * s, kc, 0, 0);
        tma_load_3d(b0 + s * bbytes, &tb, full + 8 * s, kc, nb * p.BN, 0);
      }
    } else if (warp == 1 && lane == 0) {
      for (int kt = 0; kt < p.KT; ++kt) {
        const int s = kt % p.ST;
        mbar_wait(full + 8 * s, (kt / p.ST) & 1);
        tc_fence_after();
        if (tr && kt == 0) tr[3] = gtime();
        const uint32_t sa = a0 + s * kA, sb = b0 + s * bbytes;
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          umma_bf16(tmem, sdesc(sa + kk * 32), sdesc(sb + kk * 32), p.idesc, (kt | kk) != 0);
        if (kt + p.ST < p.KT) umma_commit(empty + 8 * s);
      }
      umma_commit(done);
    }
  } else if (threadIdx.x == 32 && !(p.skip & 32)) {
    if (p.skip & 4) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(done) : "memory");
    else umma_commit(done);
  }
  if (!(p.skip & 32)) mbar_wait(done, 0);
  __syncwarp();
  tc_fence_after();
  if (tr && threadIdx.x == 0) tr[4] = gtime();
  if (p.skip & 2) goto out;
  {
    const int row = warp * 32 + lane;
    const uint32_t trow = tmem + (static_cast<uint32_t>(warp * 32) << 16);
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
    if (tr && threadIdx.x == 0) tr[5] = gtime();
    if (p.S == 1) {
      if (threadIdx.x == 0) {
        for (int c0 = 0; c0 < p.BN; c0 += 32) tma_store_3d(&tc, base + (c0 / 32) * 16384, nb * p.BN + c0, 0, 0);
        bulk_commit();
        bulk_wait_all();
      }
    } else if (p.red == 0 && (p.skip & 256)) {
      // no zeroing: the first CTA of the tile to finish stores its partial,
      // releases the tile once the store has completed; the others add
      if (threadIdx.x == 0) {
        if (tr) tr[6] = gtime();
        const uint32_t t = atomicAdd(p.cnt + tile, 1u);
        const uint32_t L = t / static_cast<uint32_t>(p.S);
        if (t % static_cast<uint32_t>(p.S) == 0) {
          for (int c0 = 0; c0 < p.BN; c0 += 32) tma_store_3d(&tc, base + (c0 / 32) * 16384, nb * p.BN + c0, 0, 0);
          bulk_commit();
          bulk_wait_all();
          fence_proxy_async_global();
          st_release_u32(p.flag + tile, L + 1);
        } else {
          while (ld_acquire_u32(p.flag + tile) < L + 1) {
          }
          fence_proxy_async_global();
          for (int c0 = 0; c0 < p.BN; c0 += 32)
            tma_reduce_add_3d(&tc, base + (c0 / 32) * 16384, nb * p.BN + c0, 0, 0);
          bulk_commit();
          bulk_wait_all();
        }
        if (tr) tr[7] = gtime();
      }
    } else if (p.red == 0) {
      if (s_ticket % static_cast<uint32_t>(p.S) != 0) {
        if (threadIdx.x == 0) {
          if (p.skip & 512) {
            while (!s_ready) {
            }
          } else {
            while (ld_acquire_u32(p.flag + tile) < s_ticket / static_cast<uint32_t>(p.S) + 1) {
            }
          }
        }
        __syncthreads();
      }
      if (threadIdx.x == 0) {
        if (tr) tr[6] = gtime();
        fence_proxy_async_global();
        for (int c0 = 0; c0 < p.BN; c0 += 32) tma_reduce_add_3d(&tc, base + (c0 / 32) * 16384, nb * p.BN + c0, 0, 0);
        bulk_commit();
        if (p.skip & 1024) bulk_wait_read();
        else bulk_wait_all();
        if (tr) tr[7] = gtime();
      }
    } else {
      // fixed-order reduction: partial -> ws[split]; arrive; every CTA of the
      // tile sums its slice of the S partials in split order
      if (threadIdx.x == 0) {
        for (int c0 = 0; c0 < p.BN; c0 += 32) tma_store_3d(&tw, base + (c0 / 32) * 16384, nb * p.BN + c0, 0, split);
        bulk_commit();
        bulk_wait_all();
        fence_proxy_async_global();
        uint32_t t;
        asm volatile("atom.add.release.gpu.global.u32 %0, [%1], 1;" : "=r"(t) : "l"(p.cnt + tile) : "memory");
        const uint32_t target = (t / p.S + 1) * p.S;
        while (ld_acquire_u32(p.cnt + tile) < target) {
        }
      }
      __syncthreads();
      const int e4 = 32 * p.BN;
      const int lo = split * e4 / p.S, hi = (split + 1) * e4 / p.S;
      const int64_t plane = 128LL * p.N;
      for (int e = lo + threadIdx.x; e < hi; e += 128) {
        const int r = e / c4, cc = (e % c4) * 4;
        const float4* src = reinterpret_cast<const float4*>(p.ws + static_cast<int64_t>(r) * p.N + nb * p.BN + cc);
        float4 acc = __ldcg(src);
        for (int s = 1; s < p.S; ++s) {
          const float4 v = __ldcg(reinterpret_cast<const float4*>(reinterpret_cast<const float*>(src) + s * plane));
          acc.x += v.x;
          acc.y += v.y;
          acc.z += v.z;
          acc.w += v.w;
        }
        *reinterpret_cast<float4*>(ctile + static_cast<int64_t>(r) * p.N + cc) = acc;
      }
    }
  }
out:
  tc_fence_before();
  __syncthreads();
  if (warp == 0 && !(p.skip & 4))
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(p.tmem_cols) : "memory");
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static EncodeTiledFn enc() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* q = nullptr;
    cudaDriverEntryPointQueryResult r;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &q, cudaEnableDefault, &r));
    fn = reinterpret_cast<EncodeTiledFn>(q);
  }
  return fn;
}
static CUtensorMap map3(void* base, CUtensorMapDataType dt, int esz, int64_t d0, int64_t d1, int64_t d2, int b0,
                        int b1) {
  CUtensorMap m;
  cuuint64_t dims[3] = {(cuuint64_t)d0, (cuuint64_t)d1, (cuuint64_t)d2};
  cuuint64_t str[2] = {(cuuint64_t)(d0 * esz), (cuuint64_t)(d0 * d1 * esz)};
  cuuint32_t box[3] = {(cuuint32_t)b0, (cuuint32_t)b1, 1};
  cuuint32_t es[3] = {1, 1, 1};
  if (enc()(&m, dt, 3, base, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
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

int main(int argc, char** argv) {
  const int M = 128, N = 768, K = 3072;
  struct V { int BN, S, CN, ST, skip; };  // ST 0: every k-tile in flight
  std::vector<V> vs;
  // launch-floor probes: 1|2 nothing, 4 no TMEM, 8 early launch_dependents, 16 no PDL, 32 no mbarriers
  for (int S : {6, 12}) {
    vs.push_back({32, S, 1, 0, 1 | 2 | 4 | 32});
    vs.push_back({32, S, 1, 0, 1 | 2 | 4 | 32 | 8});
    vs.push_back({32, S, 1, 0, 1 | 2 | 4 | 32 | 16});
    vs.push_back({32, S, 1, 0, 1 | 2 | 4});
    vs.push_back({32, S, 1, 0, 1 | 2});
    vs.push_back({32, S, 1, 0, 1 | 2 | 8});
    vs.push_back({32, S, 1, 0, 1 | 2 | 16});
    vs.push_back({32, S, 1, 2, 1 | 2});
    vs.push_back({32, S, 1, 2, 1 | 2 | 8});
  }
  vs.push_back({16, 12, 1, 0, 1 | 2 | 4 | 32});   // 576 CTAs
  vs.push_back({64, 12, 1, 0, 1 | 2 | 4 | 32});   // 144 CTAs
  vs.push_back({128, 12, 1, 0, 1 | 2 | 4 | 32});  // 72
  // full kernels: stages and early trigger
  for (int bn : {32, 64})
    for (int S : {6, 12})
      for (int st : {0, 1, 2})
        for (int sk : {0, 8, 2, 10}) vs.push_back({bn, S, 1, st, sk});
  const bool trace = argc == 7 && std::string(argv[6]) == "trace";
  if (argc == 6 || trace) {  // one variant: BN S CN ST skip [trace]
    vs.clear();
    vs.push_back({atoi(argv[1]), atoi(argv[2]), atoi(argv[3]), atoi(argv[4]), atoi(argv[5])});
  }
  if (argc == 2) {  // list the default variants
    for (const V& v : vs) printf("%d %d %d %d %d\n", v.BN, v.S, v.CN, v.ST, v.skip);
    return 0;
  }
  std::vector<uint16_t> ha(M * K), hb(N * K);
  std::vector<float> fa(M * K), fb(N * K);
  uint32_t s = 12345;
  for (int i = 0; i < M * K; ++i) {
    s = s * 1664525u + 1013904223u;
    fa[i] = static_cast<float>(static_cast<int>((s >> 24) % 5) - 2);
    ha[i] = f2bf(fa[i]);
  }
  for (int i = 0; i < N * K; ++i) {
    s = s * 1664525u + 1013904223u;
    fb[i] = static_cast<float>(static_cast<int>((s >> 24) % 5) - 2);
    hb[i] = f2bf(fb[i]);
  }
  std::vector<double> ref(M * N, 0.0);
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n) {
      double acc = 0;
      for (int k = 0; k < K; ++k) acc += static_cast<double>(fa[m * K + k]) * fb[n * K + k];
      ref[m * N + n] = acc;
    }
  void *da, *db;
  float *dc, *dws;
  uint32_t *dcnt, *dflag;
  CK(cudaMalloc(&da, ha.size() * 2));
  CK(cudaMalloc(&db, hb.size() * 2));
  CK(cudaMalloc(&dc, M * N * 4));
  CK(cudaMalloc(&dws, 64LL * M * N * 4));
  CK(cudaMalloc(&dcnt, 4096 * 4));
  CK(cudaMalloc(&dflag, 4096 * 4));
  CK(cudaMemcpy(da, ha.data(), ha.size() * 2, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(db, hb.data(), hb.size() * 2, cudaMemcpyHostToDevice));
  int optin = 0;
  CK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, 0));
  CK(cudaFuncSetAttribute(lab_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, optin - 64));
  CK(cudaFuncSetAttribute(lab_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  CUtensorMap tma_cn[5];
  for (int cn : {1, 2, 4}) tma_cn[cn] = map3(da, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, K, M, 1, 64, 128 / cn);
  CUtensorMap tmc = map3(dc, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, N, M, 1, 32, 128);
  CUtensorMap tmw = map3(dws, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, N, M, 64, 32, 128);
  cudaStream_t st;
  CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  void* scrub;
  CK(cudaMalloc(&scrub, 256 << 20));

  if (argc != 6 && !trace) printf("BN S CN ST skip ctas smemKB | graph_us iso_us exact\n");
  for (const V& v : vs) {
    P p{};
    p.N = N;
    p.K = K;
    p.BN = v.BN;
    p.S = v.S;
    p.KT = K / 64 / v.S;
    p.CN = v.CN;
    p.red = 0;
    p.ST = v.ST ? std::min(v.ST, p.KT) : p.KT;
    p.skip = v.skip;
    p.c = dc;
    p.ws = dws;
    p.cnt = dcnt;
    p.flag = dflag;
    p.idesc = (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(v.BN >> 3) << 17) |
              (static_cast<uint32_t>(128 >> 4) << 24);
    uint32_t cols = 32;
    while (cols < static_cast<uint32_t>(v.BN)) cols <<= 1;
    p.tmem_cols = cols;
    const int ring = p.ST * (kA + v.BN * 128), stgb = (v.BN / 32) * 16384;
    const int smem = 1024 + std::max(ring, stgb) + 16 * p.ST + 32;
    if (smem > optin - 64) continue;
    CUtensorMap tmb = map3(db, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, K, N, 1, 64, v.BN);
    CK(cudaMemsetAsync(dcnt, 0, 4096 * 4, st));
    CK(cudaMemsetAsync(dflag, 0, 4096 * 4, st));
    CK(cudaMemsetAsync(dc, 0xff, M * N * 4, st));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(N / v.BN, 1, v.S);
    cfg.blockDim = dim3(128);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = v.CN;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = (v.skip & 16) ? 0 : 1;
    cfg.attrs = at;
    cfg.numAttrs = 2;
    const CUtensorMap tma = tma_cn[v.CN];
    auto launch = [&]() { return cudaLaunchKernelEx(&cfg, lab_kernel, tma, tmb, tmc, tmw, p); };
    if (launch() != cudaSuccess) {
      printf("%d %d %d %d %d launch failed: %s\n", v.BN, v.S, v.CN, v.ST, v.skip, cudaGetErrorString(cudaGetLastError()));
      continue;
    }
    CK(cudaStreamSynchronize(st));
    // graph of G back-to-back launches
    const int G = 64;
    const int ctas = (N / v.BN) * v.S;
    unsigned long long* dtr = nullptr;
    if (trace) {
      CK(cudaMalloc(&dtr, sizeof(unsigned long long) * G * ctas * 9));
      CK(cudaMemset(dtr, 0, sizeof(unsigned long long) * G * ctas * 9));
    }
    cudaGraph_t g;
    cudaGraphExec_t ge;
    CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    for (int i = 0; i < G; ++i) {
      p.tr = trace ? dtr + static_cast<size_t>(i) * ctas * 9 : nullptr;
      CK(launch());
    }
    p.tr = nullptr;
    CK(cudaStreamEndCapture(st, &g));
    CK(cudaGraphInstantiate(&ge, g, 0));
    CK(cudaGraphLaunch(ge, st));
    CK(cudaStreamSynchronize(st));
    float best = 1e30f;
    std::vector<float> gt;
    for (int rep = 0; rep < 7; ++rep) {
      CK(cudaGraphLaunch(ge, st));  // keep the clocks up: the timed replay follows a busy GPU
      CK(cudaEventRecord(e0, st));
      CK(cudaGraphLaunch(ge, st));
      CK(cudaEventRecord(e1, st));
      CK(cudaEventSynchronize(e1));
      float ms;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      gt.push_back(ms * 1000.f / G);
    }
    std::sort(gt.begin(), gt.end());
    best = gt[gt.size() / 2];  // median
    if (trace) {
      std::vector<unsigned long long> h(static_cast<size_t>(G) * ctas * 9);
      CK(cudaMemcpy(h.data(), dtr, h.size() * 8, cudaMemcpyDeviceToHost));
      const char* names[8] = {"entry", "setup", "depwait", "1st k-tile", "mma done", "staged", "flag", "reduced"};
      std::vector<std::vector<double>> ph(8);
      std::vector<double> gap, span, skew;
      for (int L = 8; L < G; ++L) {
        const unsigned long long* a = &h[static_cast<size_t>(L) * ctas * 9];
        const unsigned long long* b = &h[static_cast<size_t>(L - 1) * ctas * 9];
        unsigned long long t0min = ~0ull, t0max = 0, endmax = 0, pend = 0;
        for (int c = 0; c < ctas; ++c) {
          t0min = std::min(t0min, a[9 * c]);
          t0max = std::max(t0max, a[9 * c]);
          for (int k = 0; k < 8; ++k) if (a[9 * c + k]) endmax = std::max(endmax, a[9 * c + k]);
          for (int k = 0; k < 8; ++k) if (b[9 * c + k]) pend = std::max(pend, b[9 * c + k]);
        }
        gap.push_back(static_cast<double>(t0min) - static_cast<double>(pend));
        span.push_back(static_cast<double>(endmax - t0min));
        skew.push_back(static_cast<double>(t0max - t0min));
        for (int c = 0; c < ctas; ++c)
          for (int k = 1; k < 8; ++k) {
            const unsigned long long x = a[9 * c + k], y = a[9 * c + k - 1];
            if (x && y) ph[k].push_back(static_cast<double>(x) - static_cast<double>(y));
          }
      }
      auto med = [](std::vector<double> v) { if (v.empty()) return 0.0; std::sort(v.begin(), v.end()); return v[v.size() / 2]; };
      auto p90 = [](std::vector<double> v) { if (v.empty()) return 0.0; std::sort(v.begin(), v.end()); return v[v.size() * 9 / 10]; };
      printf("trace BN %d S %d CN %d ST %d: per-launch %.2f us; span(first entry->last stamp) med %.0f ns, "
             "start skew med %.0f ns, gap(prev last stamp->first entry) med %.0f ns\n",
             v.BN, v.S, v.CN, p.ST, best, med(span), med(skew), med(gap));
      for (int k = 1; k < 8; ++k)
        printf("  %-10s -> %-10s  med %6.0f ns  p90 %6.0f ns\n", names[k - 1], names[k], med(ph[k]), p90(ph[k]));
      CK(cudaFree(dtr));
    }
    // isolated: L2 warm, one launch between events
    std::vector<float> iso;
    for (int rep = 0; rep < 15; ++rep) {
      CK(cudaEventRecord(e0, st));
      CK(launch());
      CK(cudaEventRecord(e1, st));
      CK(cudaEventSynchronize(e1));
      float ms;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      iso.push_back(ms * 1000.f);
    }
    std::sort(iso.begin(), iso.end());
    std::vector<float> hc(M * N);
    CK(cudaMemcpy(hc.data(), dc, M * N * 4, cudaMemcpyDeviceToHost));
    bool exact = true;
    for (int i = 0; i < M * N && exact; ++i) exact = static_cast<double>(hc[i]) == ref[i];
    if (v.skip & 3 & ~64) exact = true;
    printf("%3d %2d %d %d %2d %3d %5.1f | %6.2f %6.2f %s\n", v.BN, v.S, v.CN, p.ST, v.skip, (N / v.BN) * v.S,
           smem / 1024.0, best, iso[iso.size() / 2], exact ? "exact" : "MISMATCH");
    fflush(stdout);
    CK(cudaGraphExecDestroy(ge));
    CK(cudaGraphDestroy(g));
  }
  return 0;
}
