// GEMM lab 2: "units per CTA" -- each CTA of a split-K tcgen05 GEMM processes
// U work units (tile x split) back to back: one launch floor for half the
// CTAs, and the epilogue of unit j (warps 0-3: TMEM -> smem -> TMA add-reduce)
// overlaps the loads / MMAs of unit j+1 (warp 4: TMA producer + split-K
// tickets, warp 5: MMA issuer).  BERT FFN 128x768x3072, mode-2 reduction
// (ticket + in-kernel zeroing), BN % 32 == 0.  Exactness checked on
// small-integer inputs; per-launch time from CUDA graphs of 64 PDL launches,
// median of 7 interleaved rounds.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 scripts/gemm_lab2.cu -o /tmp/gemm_lab2 -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

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

constexpr int kA = 128 * 64 * 2;
constexpr int kMaxU = 4;

struct P {
  int N, BN, S, KT, ST, U, units;  // units = tiles x splits
  float* c;
  uint32_t* cnt;
  uint32_t* flag;
  uint32_t idesc, cols;  // cols: TMEM columns per accumulator (power of 2 >= BN)
  uint32_t alloc;        // TMEM columns allocated: power of 2 >= cols * U
};

__global__ void __launch_bounds__(192, 1)
lab2(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb,
     const __grid_constant__ CUtensorMap tc, P p) {
  extern __shared__ uint8_t smem_raw[];
  __shared__ uint32_t s_ticket[kMaxU];
  __shared__ uint32_t s_slot;
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* gbase = smem_raw + (base - raw);
  const int bbytes = p.BN * 128;
  const uint32_t a0 = base, b0 = base + p.ST * kA;
  const uint32_t stg = b0 + p.ST * bbytes;  // epilogue staging, separate from the ring
  const uint32_t stg_bytes = static_cast<uint32_t>(p.BN / 32) * 16384u;
  const uint32_t bars = stg + stg_bytes;
  const uint32_t full = bars, empty = bars + 8 * p.ST, done = bars + 16 * p.ST;  // done[U]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tiles = p.N / p.BN;
  int nunits = 0;
  int uidx[kMaxU];
  for (int j = 0; j < p.U; ++j) {
    const int u = blockIdx.x + j * gridDim.x;
    if (u < p.units) uidx[nunits++] = u;
  }

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&s_slot)),
                 "r"(p.alloc)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (threadIdx.x == 32) {
    for (int s = 0; s < p.ST; ++s) {
      mbar_init(full + 8 * s, 1);
      mbar_init(empty + 8 * s, 1);
    }
    for (int j = 0; j < p.U; ++j) mbar_init(done + 8 * j, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&ta)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tb)) : "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = s_slot;
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");

  if (warp == 4) {
    // split-K tickets of every unit; the tile's first arriver zeroes it
    if (lane < nunits) s_ticket[lane] = atomicAdd(p.cnt + uidx[lane] % tiles, 1u);
    __syncwarp();
    for (int j = 0; j < nunits; ++j) {
      const uint32_t t = s_ticket[j];
      if (t % static_cast<uint32_t>(p.S) != 0) continue;
      const int tile = uidx[j] % tiles;
      float* ct = p.c + static_cast<int64_t>(tile) * p.BN;
      const int c4 = p.BN / 4;
      const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int e = lane; e < 128 * c4; e += 32)
        *reinterpret_cast<float4*>(ct + static_cast<int64_t>(e / c4) * p.N + (e % c4) * 4) = z;
      __syncwarp();
      if (lane == 0) st_release_u32(p.flag + tile, t / p.S + 1);
    }
    if (lane == 0) {  // ---- TMA producer over every unit's k-tiles ----
      int g = 0;
      for (int j = 0; j < nunits; ++j) {
        const int tile = uidx[j] % tiles, split = uidx[j] / tiles;
        for (int kt = 0; kt < p.KT; ++kt, ++g) {
          const int s = g % p.ST;
          if (g >= p.ST) mbar_wait(empty + 8 * s, ((g / p.ST) & 1) ^ 1);
          const int kc = (split * p.KT + kt) * 64;
          mbar_expect_tx(full + 8 * s, kA + bbytes);
          tma_load_3d(a0 + s * kA, &ta, full + 8 * s, kc, 0, 0);
          tma_load_3d(b0 + s * bbytes, &tb, full + 8 * s, kc, tile * p.BN, 0);
        }
      }
    }
  } else if (warp == 5) {
    if (lane == 0) {  // ---- MMA issuer ----
      int g = 0;
      for (int j = 0; j < nunits; ++j) {
        const uint32_t acc = tmem + static_cast<uint32_t>(j) * p.cols;
        for (int kt = 0; kt < p.KT; ++kt, ++g) {
          const int s = g % p.ST;
          mbar_wait(full + 8 * s, (g / p.ST) & 1);
          tc_fence_after();
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            umma_bf16(acc, sdesc(a0 + s * kA + kk * 32), sdesc(b0 + s * bbytes + kk * 32), p.idesc, (kt | kk) != 0);
          umma_commit(empty + 8 * s);
        }
        umma_commit(done + 8 * j);
      }
    }
  } else {
    // ---- epilogue, warps 0-3 (TMEM lanes 32w..32w+31 = output rows) ----
    const int row = warp * 32 + lane;
    for (int j = 0; j < nunits; ++j) {
      mbar_wait(done + 8 * j, 0);
      __syncwarp();
      tc_fence_after();
      const uint32_t trow = tmem + static_cast<uint32_t>(j) * p.cols + (static_cast<uint32_t>(warp * 32) << 16);
      if (j > 0 && threadIdx.x == 0) bulk_wait_read();  // the previous unit's staging has been read
      asm volatile("bar.sync 1, 128;" ::: "memory");
      for (int c0 = 0; c0 < p.BN; c0 += 32) {
        uint32_t v[32];
        tmem_ld16_nowait(trow + c0, v);
        tmem_ld16_nowait(trow + c0 + 16, v + 16);
        tmem_wait();
        uint8_t* chunk = gbase + (stg - base) + (c0 / 32) * 16384 + row * 128;
#pragma unroll
        for (int q = 0; q < 8; ++q)
          *reinterpret_cast<float4*>(chunk + ((q ^ (row & 7)) << 4)) =
              make_float4(__uint_as_float(v[4 * q]), __uint_as_float(v[4 * q + 1]), __uint_as_float(v[4 * q + 2]),
                          __uint_as_float(v[4 * q + 3]));
      }
      fence_proxy_async_smem();
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (threadIdx.x == 0) {
        const int tile = uidx[j] % tiles;
        const uint32_t t = s_ticket[j];
        if (t % static_cast<uint32_t>(p.S) != 0) {
          uint32_t spins = 0;
          while (ld_acquire_u32(p.flag + tile) < t / static_cast<uint32_t>(p.S) + 1)
            if (++spins > (1u << 26)) __trap();
        }
        fence_proxy_async_global();
        for (int c0 = 0; c0 < p.BN; c0 += 32) tma_reduce_add_3d(&tc, stg + (c0 / 32) * 16384, tile * p.BN + c0, 0, 0);
        bulk_commit();
      }
    }
    if (threadIdx.x == 0) bulk_wait_all();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(p.alloc) : "memory");
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static CUtensorMap map3(void* base, CUtensorMapDataType dt, int esz, int64_t d0, int64_t d1, int b0, int b1) {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* q = nullptr;
    cudaDriverEntryPointQueryResult r;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &q, cudaEnableDefault, &r));
    fn = reinterpret_cast<EncodeTiledFn>(q);
  }
  CUtensorMap m;
  cuuint64_t dims[3] = {(cuuint64_t)d0, (cuuint64_t)d1, 1};
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
  const int M = 128, N = 768, K = 3072;
  std::vector<uint16_t> ha(M * K), hb(N * K);
  std::vector<float> fa(M * K), fb(N * K);
  uint32_t s = 777;
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
  float* dc;
  uint32_t *dcnt, *dflag;
  CK(cudaMalloc(&da, ha.size() * 2));
  CK(cudaMalloc(&db, hb.size() * 2));
  CK(cudaMalloc(&dc, M * N * 4));
  CK(cudaMalloc(&dcnt, 4096 * 4));
  CK(cudaMalloc(&dflag, 4096 * 4));
  CK(cudaMemcpy(da, ha.data(), ha.size() * 2, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(db, hb.data(), hb.size() * 2, cudaMemcpyHostToDevice));
  int optin = 0;
  CK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, 0));
  CK(cudaFuncSetAttribute(lab2, cudaFuncAttributeMaxDynamicSharedMemorySize, optin - 1024));
  CUtensorMap tma = map3(da, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, K, M, 64, 128);
  CUtensorMap tmc = map3(dc, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, N, M, 32, 128);
  cudaStream_t st;
  CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  struct V {
    int BN, S, U, ST;
  };
  std::vector<V> vs;
  for (int bn : {32, 64, 96})
    for (int S : {6, 8, 12, 16, 24})
      for (int U : {1, 2, 3}) {
        const int KT = 48 / S;
        if (48 % S || KT < 1) continue;
        const int units = (N / bn) * S;
        if (units / U > 300 || units / U < 60) continue;
        vs.push_back({bn, S, U, std::min(KT * U, 8)});
      }
  std::vector<cudaGraphExec_t> ge(vs.size());
  std::vector<std::vector<float>> t(vs.size());
  std::vector<int> ok(vs.size(), 0), grid(vs.size(), 0), smemv(vs.size(), 0);
  const int G = 64;
  for (size_t i = 0; i < vs.size(); ++i) {
    const V& v = vs[i];
    P p{};
    p.N = N;
    p.BN = v.BN;
    p.S = v.S;
    p.KT = 48 / v.S;
    p.ST = v.ST;
    p.U = v.U;
    p.units = (N / v.BN) * v.S;
    p.c = dc;
    p.cnt = dcnt;
    p.flag = dflag;
    p.idesc = (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(v.BN >> 3) << 17) |
              (static_cast<uint32_t>(128 >> 4) << 24);
    uint32_t cols = 32;
    while (cols < static_cast<uint32_t>(v.BN)) cols <<= 1;
    p.cols = cols;
    p.alloc = 32;
    while (p.alloc < cols * v.U) p.alloc <<= 1;
    if (p.alloc > 512) continue;
    const int smem = 1024 + p.ST * (kA + v.BN * 128) + (v.BN / 32) * 16384 + 16 * p.ST + 8 * v.U + 64;
    if (smem > optin - 1024) continue;
    CUtensorMap tmb = map3(db, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, K, N, 64, v.BN);
    CK(cudaStreamSynchronize(st));  // the previous variant's graph ran on st (non-blocking)
    const int per_sm = std::min(optin / smem, 512 / static_cast<int>(p.alloc));
    if (per_sm * 148 < (p.units + v.U - 1) / v.U) continue;  // split-K flags need co-residency
    CK(cudaMemset(dcnt, 0, 4096 * 4));
    CK(cudaMemset(dflag, 0, 4096 * 4));
    cudaLaunchConfig_t cfg = {};
    grid[i] = (p.units + v.U - 1) / v.U;
    smemv[i] = smem;
    cfg.gridDim = dim3(grid[i]);
    cfg.blockDim = dim3(192);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    CK(cudaMemset(dc, 0xff, M * N * 4));
    CK(cudaLaunchKernelEx(&cfg, lab2, tma, tmb, tmc, p));
    CK(cudaStreamSynchronize(st));
    fprintf(stderr, "variant BN%d S%d U%d launched ok\n", v.BN, v.S, v.U);
    std::vector<float> hc(M * N);
    CK(cudaMemcpy(hc.data(), dc, M * N * 4, cudaMemcpyDeviceToHost));
    bool exact = true;
    for (int k = 0; k < M * N && exact; ++k) exact = static_cast<double>(hc[k]) == ref[k];
    ok[i] = exact;
    cudaGraph_t g;
    CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    for (int k = 0; k < G; ++k) CK(cudaLaunchKernelEx(&cfg, lab2, tma, tmb, tmc, p));
    CK(cudaStreamEndCapture(st, &g));
    CK(cudaGraphInstantiate(&ge[i], g, 0));
    CK(cudaGraphLaunch(ge[i], st));
  }
  CK(cudaStreamSynchronize(st));
  for (int r = 0; r < 7; ++r)
    for (size_t i = 0; i < vs.size(); ++i) {
      if (!ge[i]) continue;
      CK(cudaGraphLaunch(ge[i], st));
      CK(cudaEventRecord(e0, st));
      CK(cudaGraphLaunch(ge[i], st));
      CK(cudaEventRecord(e1, st));
      CK(cudaEventSynchronize(e1));
      float ms;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      t[i].push_back(ms * 1000.f / G);
    }
  printf("BN S U ST ctas smemKB | median_us exact\n");
  for (size_t i = 0; i < vs.size(); ++i) {
    if (!ge[i]) continue;
    std::sort(t[i].begin(), t[i].end());
    printf("%3d %2d %d %d %3d %5.1f | %6.2f %s\n", vs[i].BN, vs[i].S, vs[i].U, vs[i].ST, grid[i], smemv[i] / 1024.0,
           t[i][3], ok[i] ? "exact" : "MISMATCH");
  }
  return 0;
}
