// The B200 Runner: instantiate each candidate program as a kernel, run it,
// check its output against the e0 reference output (K6) and time it with CUDA
// events -- the hardware replacement of `_measure_batch`
// (`src/search.py:249-256`) and of the baseline `simulate_latency(e0)`
// (`src/search.py:326`).
//
// Timing protocol per ls_runner_measure call:
//   phase A  (checked run)  for every launchable candidate: poison C with NaN,
//            zero it when the family accumulates, arm a device-side deadline,
//            launch once, run the parity reducer.  One sync for the batch.
//   phase B  (timed run)    repeats sized from phase A (target_ms), launched
//            back to back between two events per candidate.  Launches are
//            queued in chunks behind a short device spin so the host has
//            enqueued a whole chunk before its first event fires: the events
//            bracket device execution, never host launch gaps.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <climits>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "../../include/loopsched_b200.h"
#include "common.hpp"
#include "ir.hpp"
#include "affine.hpp"
#include "generic.cuh"
#include "kernels.cuh"
#include "plan.hpp"
#include "simta.cuh"
#include "tc_conv.cuh"

using namespace lsb;

namespace {

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

// K-major operand [batch][rows][K] as a 3-D TMA map whose box is one
// 128-byte swizzle row per operand row: {64, box_rows, 1} of bf16, or
// {32, box_rows, 1} of fp32 (the 3xTF32 halves; batch then counts hi and lo).
bool make_kmajor_map(CUtensorMap* map, void* base, int64_t batch, int64_t rows, int64_t k, int box_rows,
                     bool f32 = false) {
  EncodeTiledFn enc = encode_fn();
  if (!enc) return false;
  const int64_t es = f32 ? 4 : 2;
  cuuint64_t dims[3] = {static_cast<cuuint64_t>(k), static_cast<cuuint64_t>(rows), static_cast<cuuint64_t>(batch)};
  cuuint64_t strides[2] = {static_cast<cuuint64_t>(k * es), static_cast<cuuint64_t>(rows * k * es)};
  cuuint32_t box[3] = {static_cast<cuuint32_t>(128 / es), static_cast<cuuint32_t>(box_rows), 1};
  cuuint32_t estr[3] = {1, 1, 1};
  return enc(map, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, base, dims, strides,
             box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// fp32 output [batch][M][N] as a 3-D TMA map with a {32, 128, 1} box and the
// 128-byte swizzle (the tcgen05 epilogue's staged chunk layout).
bool make_c_map(CUtensorMap* map, void* base, int64_t batch, int64_t m, int64_t n) {
  EncodeTiledFn enc = encode_fn();
  if (!enc || n % 4 != 0) return false;
  cuuint64_t dims[3] = {static_cast<cuuint64_t>(n), static_cast<cuuint64_t>(m), static_cast<cuuint64_t>(batch)};
  cuuint64_t strides[2] = {static_cast<cuuint64_t>(n * 4), static_cast<cuuint64_t>(m * n * 4)};
  cuuint32_t box[3] = {32, 128, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, base, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
             CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// fp32 NHWC output [n][p][q][k] as a 4-D TMA map with a {32, 8, 8, 1} box and
// the 128-byte swizzle (the tcgen05 conv epilogue's staged chunk layout).
bool make_nhwc_out_map(CUtensorMap* map, void* base, const int64_t* shape) {
  EncodeTiledFn enc = encode_fn();
  if (!enc || shape[3] % 4 != 0) return false;
  cuuint64_t dims[4] = {static_cast<cuuint64_t>(shape[3]), static_cast<cuuint64_t>(shape[2]),
                        static_cast<cuuint64_t>(shape[1]), static_cast<cuuint64_t>(shape[0])};
  cuuint64_t strides[3] = {static_cast<cuuint64_t>(shape[3] * 4), static_cast<cuuint64_t>(shape[2] * shape[3] * 4),
                           static_cast<cuuint64_t>(shape[1] * shape[2] * shape[3] * 4)};
  cuuint32_t box[4] = {32, 8, 8, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, base, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
             CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// NHWC activation [n][h][w][c] as a 4-D TMA map whose box is one 8 x 8 pixel
// box of 128-byte channel rows: {64, 8, 8, 1} of bf16, or {32, 8, 8, 1} of
// fp32 over the [hi | lo] halves of the 3xTF32 tile (n doubled, lo at n + N);
// out-of-bounds boxes read zeros.
bool make_nhwc_map(CUtensorMap* map, void* base, const int64_t* shape, bool f32 = false) {
  EncodeTiledFn enc = encode_fn();
  if (!enc) return false;
  const int64_t es = f32 ? 4 : 2;
  cuuint64_t dims[4] = {static_cast<cuuint64_t>(shape[3]), static_cast<cuuint64_t>(shape[2]),
                        static_cast<cuuint64_t>(shape[1]), static_cast<cuuint64_t>(shape[0] * (f32 ? 2 : 1))};
  cuuint64_t strides[3] = {static_cast<cuuint64_t>(shape[3] * es), static_cast<cuuint64_t>(shape[2] * shape[3] * es),
                           static_cast<cuuint64_t>(shape[1] * shape[2] * shape[3] * es)};
  cuuint32_t box[4] = {static_cast<cuuint32_t>(128 / es), 8, 8, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  return enc(map, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, base, dims, strides,
             box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
             CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

void fill_result(const Plan& p, ls_result* r) {
  std::memset(r, 0, sizeof *r);
  r->family = p.family;
  r->status = p.status == P_OK ? LS_RUN_OK
            : p.status == P_ILLEGAL ? LS_RUN_ILLEGAL
            : p.status == P_PARSE ? LS_RUN_PARSE
            : LS_RUN_UNSUPPORTED;
  std::memcpy(r->cfg, p.cfg, sizeof r->cfg);
}

}  // namespace

// checked-launch gates (phase A): candidates per gated chunk, safety timeout
constexpr int kGateChunk = 16;
constexpr unsigned long long kGateMaxNs = 2000000ull;  // a chunk enqueues in ~0.3 ms; serialised launches (profilers) pay <= 2 ms per gate

struct ls_runner {
  int device = 0;
  ls_runner_opts opts{};
  cudaStream_t st = nullptr;
  bool bf16 = false;
  bool have_workload = false;
  bool best_valid = false;  // device best-so-far initialised for this workload (carry_best)
  int64_t setup_launches = 0;  // kernels of the last set_workload, reported by the next measure call's count
  Workload w;
  std::string e0_text;
  bool tc_ok = false;
  void* x = nullptr;        // device inputs in the runner dtype
  void* y = nullptr;
  void* yk = nullptr;       // K-major copy of Y for the tcgen05 family (bf16; fp32: [hi | lo] halves)
  void* xs = nullptr;       // fp32 workloads: [hi | lo] halves of X for the 3xTF32 tcgen05 tile
  float* c = nullptr;
  double* ref = nullptr;
  Strides s{};
  CUtensorMap tmap_a{};
  CUtensorMap tmap_c{};
  bool have_tmap_c = false;
  std::mutex map_mu;  // tensor-map caches: phase-B graphs are captured on a helper thread
  std::map<int, CUtensorMap> tmap_am;  // A maps by box rows (TMA multicast slices)
  std::map<int, CUtensorMap> tmap_b;
  unsigned long long* deadline = nullptr;  // device deadline state: [0] deadline, [1] arm time, [2] best ns
  void* scrub = nullptr;  // flush_l2: 256 MB written before every timed repeat (L2 is 126 MB)
  static constexpr size_t kScrubBytes = 256ull << 20;
  int* flags = nullptr;                    // per-candidate timeout flags
  unsigned long long* parity = nullptr;    // per-candidate (max err bits, mismatches)
  int cap = 0;
  std::vector<cudaEvent_t> ev;             // 4 per candidate slot
  float last_ms = 0.f;
  std::atomic<int64_t> launches{0};
  unsigned int* gate = nullptr;  // mapped pinned word released by the host (launch_gate)
  unsigned int gate_seq = 0;
  void open_gate(unsigned int v) { __atomic_store_n(gate, v, __ATOMIC_RELEASE); }
  cudaStream_t cap_st = nullptr;  // phase-B graph capture on the helper thread (never executes)
  double stats[8] = {0};  // host ms phase A, phase B, spin us, plan ms, empty us, best us, phase-A enqueue ms
  DeviceLimits lim;
  double launch_host_us = 4.0;  // host enqueue cost per call, for sizing the device spin
  unsigned long long empty_ns = 0;  // device elapsed of an empty candidate (arm -> stamp), calibrated

  // Device memory pool for per-workload buffers: set_workload is called once
  // per task (and per bench step); reusing same-size blocks avoids
  // cudaMalloc/cudaFree (implicitly synchronising, ~ms) on every call.
  std::multimap<size_t, void*> pool_free;
  std::map<void*, size_t> pool_size;
  cudaError_t pmalloc(void** p, size_t n) {
    n = (n + 255) & ~static_cast<size_t>(255);
    auto it = pool_free.lower_bound(n);
    if (it != pool_free.end() && it->first <= 2 * n) {
      *p = it->second;
      pool_free.erase(it);
      return cudaSuccess;
    }
    cudaError_t e = cudaMalloc(p, n);
    if (e == cudaSuccess) pool_size[*p] = n;
    return e;
  }
  void pfree(void* p) {
    if (!p) return;
    auto it = pool_size.find(p);
    if (it == pool_size.end()) { cudaFree(p); return; }
    pool_free.emplace(it->second, p);
  }
  void pool_release() {
    for (auto& kv : pool_size) cudaFree(kv.first);
    pool_size.clear();
    pool_free.clear();
  }

  ~ls_runner() { release(); }

  void release_workload() {
    if (general)  // (the alt view of a contraction workload aliases x, y, c)
      for (size_t i = 0; i < gbuf.size(); ++i)
        if (gbuf[i] != c) pfree(gbuf[i]);
    gbuf.clear();
    has_alt = false;
    pfree(wt);
    wt = nullptr;
    for (void* h : gbuf_x3) pfree(h);
    gbuf_x3.clear();
    tmap_wt.clear();
    tmap_x.clear();
    tmap_o.clear();
    gbuf_dtype.clear();
    general = false;
    pfree(x); pfree(y); pfree(yk); pfree(xs); pfree(c); pfree(ref);
    x = y = yk = xs = nullptr; c = nullptr; ref = nullptr;
    tmap_b.clear();
    tmap_am.clear();
    have_tmap_c = false;
    have_workload = false;
    setup_launches = 0;
  }
  void release() {
    cudaSetDevice(device);
    if (st) cudaStreamSynchronize(st);
    release_workload();
    cudaFree(deadline); cudaFree(flags); cudaFree(parity); cudaFree(gcode); cudaFree(tcsync);
    cudaFree(scrub);
    scrub = nullptr;
    pool_release();
    gcode = nullptr;
    tcsync = nullptr;
    tcsync_cap = 0;
    deadline = nullptr; flags = nullptr; parity = nullptr;
    for (cudaEvent_t e : ev) cudaEventDestroy(e);
    ev.clear();
    if (st) cudaStreamDestroy(st);
    if (cap_st) cudaStreamDestroy(cap_st);
    if (gate) cudaFreeHost(gate);
    gate = nullptr;
    cap_st = nullptr;
    st = nullptr;
  }

  ls_status ensure_capacity(int n) {
    if (n <= cap) return LS_OK;
    int nc = std::max(n, 2 * cap);
    cudaFree(flags);
    cudaFree(parity);
    flags = nullptr;
    parity = nullptr;
    LSB_CUDA(cudaMalloc(&flags, static_cast<size_t>(nc) * sizeof(int)));
    LSB_CUDA(cudaMalloc(&parity, static_cast<size_t>(nc) * 2 * sizeof(unsigned long long)));
    while (ev.size() < static_cast<size_t>(nc) * 4) {
      cudaEvent_t e;
      LSB_CUDA(cudaEventCreate(&e));
      ev.push_back(e);
    }
    cap = nc;
    return LS_OK;
  }

  const CUtensorMap* map_a(int rows) {
    if (rows == 128) return &tmap_a;
    std::lock_guard<std::mutex> lk(map_mu);
    auto it = tmap_am.find(rows);
    if (it != tmap_am.end()) return &it->second;
    CUtensorMap m;
    const int64_t halves = bf16 ? 1 : 2;
    if (!make_kmajor_map(&m, bf16 ? x : xs, halves * w.extent[R_BATCH], w.extent[R_M], w.extent[R_K], rows, !bf16))
      return nullptr;
    return &(tmap_am[rows] = m);
  }
  const CUtensorMap* map_b(int bn) {
    std::lock_guard<std::mutex> lk(map_mu);
    auto it = tmap_b.find(bn);
    if (it != tmap_b.end()) return &it->second;
    CUtensorMap m;
    const int64_t halves = bf16 ? 1 : 2;
    if (!make_kmajor_map(&m, yk, halves * w.extent[R_BATCH], w.extent[R_N], w.extent[R_K], bn, !bf16)) return nullptr;
    return &(tmap_b[bn] = m);
  }

  // one launch of a planned candidate (plus its zeroing memset)
  unsigned long long* trace = nullptr;  // set only by ls_runner_trace_tc
  // split-K ticket slots (tc_geom mode 2): 2 x kTcSyncSlots words per such
  // candidate of the current call, zeroed before its first launch
  uint32_t* tcsync = nullptr;
  size_t tcsync_cap = 0;  // words
  std::vector<int64_t> sync_off;  // per candidate slot: word offset or -1

  ls_status prepare_sync(const std::vector<Plan>& plans) {
    sync_off.assign(plans.size(), -1);
    size_t words = 0;
    for (size_t i = 0; i < plans.size(); ++i) {
      const Plan& p = plans[i];
      if (p.status != P_OK) continue;
      if (p.gp) {  // tcgen05 conv step with split-K: mode 2 in tc_conv.cu
        bool want = false;
        for (const GStep& stp : p.gp->steps)
          want |= stp.family == F_TCCONV && stp.conv.splits > 1 && stp.conv.grid_m * stp.conv.grid_n <= kTcSyncSlots;
        if (!want) continue;
      } else {
        if (p.family != F_TC) continue;
        if (tc_geom(p.tc.bn, p.tc.splits, p.tc.stages, p.tc.batch * p.tc.grid_m * p.tc.grid_n, p.tc.x3).mode != 2)
          continue;
      }
      sync_off[i] = static_cast<int64_t>(words);
      words += 2 * kTcSyncSlots;
    }
    if (!words) return LS_OK;
    if (words > tcsync_cap) {
      cudaFree(tcsync);
      tcsync = nullptr;
      tcsync_cap = std::max(words, 2 * tcsync_cap);
      LSB_CUDA(cudaMalloc(&tcsync, tcsync_cap * 4));
    }
    LSB_CUDA(cudaMemsetAsync(tcsync, 0, words * 4, st));
    return LS_OK;
  }
  // general workloads (multi-block / affine contraction)
  bool general = false;
  bool has_alt = false;  // contraction workload with a general-path view in gw / gbuf (plan_all alt)
  GeneralWorkload gw;
  std::vector<void*> gbuf;      // device buffer per e0 buffer (gw.buffers order)
  std::vector<int> gbuf_dtype;  // 0 bf16, 1 f32
  int64_t* gcode = nullptr;     // concatenated bytecode of the current batch
  size_t gcode_cap = 0;
  // tcgen05 conv: K-major weight copy [n_cols][k_rows] and tensor-map caches
  void* wt = nullptr;            // bf16; fp32 workloads: [hi | lo] halves (3xTF32)
  int64_t wt_rows = 0, wt_cols = 0;
  std::vector<void*> gbuf_x3;    // fp32 workloads: [hi | lo] halves of each NHWC buffer (or null)
  std::map<int, CUtensorMap> tmap_wt;         // by BN
  std::map<const void*, CUtensorMap> tmap_x;  // by activation buffer

  const CUtensorMap* map_wt(int bn) {
    std::lock_guard<std::mutex> lk(map_mu);
    auto it = tmap_wt.find(bn);
    if (it != tmap_wt.end()) return &it->second;
    CUtensorMap m;
    if (!wt || !make_kmajor_map(&m, wt, bf16 ? 1 : 2, wt_cols, wt_rows, bn, !bf16)) return nullptr;
    return &(tmap_wt[bn] = m);
  }
  std::map<const void*, CUtensorMap> tmap_o;  // fp32 NHWC conv outputs, box {32, 8, 8, 1}
  const CUtensorMap* map_o(const void* buf, const int64_t* shape) {
    std::lock_guard<std::mutex> lk(map_mu);
    auto it = tmap_o.find(buf);
    if (it != tmap_o.end()) return &it->second;
    CUtensorMap m;
    if (!make_nhwc_out_map(&m, const_cast<void*>(buf), shape)) return nullptr;
    return &(tmap_o[buf] = m);
  }
  const CUtensorMap* map_x(const void* buf, const int64_t* shape) {
    std::lock_guard<std::mutex> lk(map_mu);
    auto it = tmap_x.find(buf);
    if (it != tmap_x.end()) return &it->second;
    CUtensorMap m;
    if (!make_nhwc_map(&m, const_cast<void*>(buf), shape, !bf16)) return nullptr;
    return &(tmap_x[buf] = m);
  }

  bool general_buffers(const Plan& p, GenBuffers* B) {
    const GenProgram& g = p.gp->gen;
    std::memset(B, 0, sizeof *B);
    for (int b = 0; b < g.nbuf; ++b) {
      const std::string& nm = p.gp->buf_names[static_cast<size_t>(b)];
      auto it = std::find(gw.buffers.begin(), gw.buffers.end(), nm);
      if (it == gw.buffers.end()) return false;
      size_t i = static_cast<size_t>(it - gw.buffers.begin());
      B->ptr[b] = gbuf[i];
      B->dtype[b] = gbuf_dtype[i];
      for (int d = 0; d < g.ndim[b]; ++d) B->shape[b][d] = g.shape[b][d];
    }
    return true;
  }

  bool launch_general(const Plan& p, const unsigned long long* dl, int* flag, int slot, cudaStream_t q) {
    GenBuffers B;
    if (!general_buffers(p, &B)) return false;
    for (const GStep& stp : p.gp->steps) {
      GenBlock g = p.gp->gen.blocks[static_cast<size_t>(stp.block)];
      bool ok = true;
      if (stp.family == F_TCCONV) {
        if (p.gp->gen.ndim[stp.x_buf] != 4 || B.dtype[stp.x_buf] != (stp.conv.x3 ? 1 : 0)) return false;
        const void* xsrc = B.ptr[stp.x_buf];
        if (stp.conv.x3) {  // the activation's [hi | lo] halves (an input's: split at set_workload)
          auto it = std::find(gw.buffers.begin(), gw.buffers.end(), p.gp->buf_names[static_cast<size_t>(stp.x_buf)]);
          const size_t gi = static_cast<size_t>(it - gw.buffers.begin());
          if (it == gw.buffers.end() || gi >= gbuf_x3.size() || !gbuf_x3[gi]) return false;
          xsrc = gbuf_x3[gi];
          if (stp.x3_split) {  // the activation was written by an earlier step of this launch
            const int64_t* sh = B.shape[stp.x_buf];
            launch_split_tf32(static_cast<const float*>(B.ptr[stp.x_buf]), static_cast<float*>(gbuf_x3[gi]), 1,
                              sh[0] * sh[1] * sh[2], sh[3], false, q);
          }
        }
        const CUtensorMap* mx = map_x(xsrc, B.shape[stp.x_buf]);
        const CUtensorMap* mw = map_wt(static_cast<int>(stp.conv.bn));
        if (!mx || !mw) return false;
        uint32_t* sy = slot >= 0 && static_cast<size_t>(slot) < sync_off.size() && sync_off[static_cast<size_t>(slot)] >= 0
                           ? tcsync + sync_off[static_cast<size_t>(slot)]
                           : nullptr;
        const CUtensorMap* mc = p.gp->gen.ndim[stp.c_buf] == 4 && B.dtype[stp.c_buf] == 1
                                    ? map_o(B.ptr[stp.c_buf], B.shape[stp.c_buf])
                                    : nullptr;
        ok = launch_tc_conv(mx, mw, static_cast<float*>(B.ptr[stp.c_buf]), stp.conv, true, q, trace, sy, mc,
                            mc ? B.shape[stp.c_buf] : nullptr, static_cast<int>(B.shape[stp.x_buf][0]));
      } else if (stp.family == F_AFFCOPY) {
        ok = launch_affcopy(stp.copy, B, dl, flag, q);
      } else if (stp.family == F_SIMTA) {
        ok = launch_simta(B.ptr[stp.x_buf], B.ptr[stp.y_buf], static_cast<float*>(B.ptr[stp.c_buf]), stp.aff, bf16, dl,
                          flag, q);
      } else if (stp.family == F_NESTGEN) {
        ok = launch_generic_nest(g, p.gcode, B, dl, flag, q);
      } else {
        if (stp.epilogue_pass) {  // rewrite the accumulated element through the epilogue
          for (int i = 0; i < g.nl; ++i)
            if ((g.red_mask >> i) & 1u) g.ext[i] = 1;
          g.red_mask = 0;
          g.red_trip = 1;
          g.value_code = g.epi_code;
          g.init_code = -1;
          g.epi_code = -1;
        }
        ok = launch_generic_block(g, p.gcode, B, false, dl, flag, q);
      }
      if (!ok) return false;
    }
    return true;
  }

  bool launch(const Plan& p, bool guarded, int slot, cudaStream_t q = nullptr) {
    if (!q) q = st;
    const unsigned long long* dl = guarded ? deadline : nullptr;
    int* flag = flags + slot;
    if (p.gp) {
      launches += general_kernels(*p.gp);
      return launch_general(p, dl, flag, slot, q);
    }
    const size_t cbytes = static_cast<size_t>(w.c_elems) * sizeof(float);
    if (p.needs_zero && cudaMemsetAsync(c, 0, cbytes, q) != cudaSuccess) return false;
    ++launches;
    switch (p.family) {
      case F_NAIVE:
        launch_naive(x, y, c, s, bf16, q);
        return cudaGetLastError() == cudaSuccess;
      case F_SIMT:
        return launch_simt(x, y, c, s, p.simt, bf16, dl, flag, q);
      case F_LOOPNEST:
        launch_loopnest(x, y, c, p.nest, bf16, dl, flag, q);
        return cudaGetLastError() == cudaSuccess;
      case F_TC: {
        const CUtensorMap* mb = map_b(static_cast<int>(p.tc.bn));
        if (!mb) return false;
        TcLaunch L;
        const CUtensorMap* ma = map_a(128);
        if (!ma) return false;
        L.tmap_a = ma;
        L.tmap_b = mb;
        L.tmap_c = have_tmap_c ? &tmap_c : nullptr;
        L.c = c;
        L.sc_b = w.sc[R_BATCH];
        L.sc_m = w.sc[R_M];
        L.m = static_cast<int>(w.extent[R_M]);
        L.n = static_cast<int>(w.extent[R_N]);
        L.k = static_cast<int>(w.extent[R_K]);
        L.bn = static_cast<int>(p.tc.bn);
        L.splits = static_cast<int>(p.tc.splits);
        L.kt = static_cast<int>(p.tc.kt);
        L.stages = static_cast<int>(p.tc.stages);
        L.batch = static_cast<int>(p.tc.batch);
        L.grid_m = static_cast<int>(p.tc.grid_m);
        L.grid_n = static_cast<int>(p.tc.grid_n);
        L.smem_bytes = static_cast<int>(p.tc.smem_bytes);
        L.trace = trace;
        L.x3 = p.tc.x3;
        L.sync = slot >= 0 && static_cast<size_t>(slot) < sync_off.size() && sync_off[static_cast<size_t>(slot)] >= 0
                     ? tcsync + sync_off[static_cast<size_t>(slot)]
                     : nullptr;
        return launch_tc_gemm(L, q);
      }
      default:
        return false;
    }
  }
};

namespace {

// kernels one Runner::launch of a plan enqueues (as counted in launches)
int64_t kernels_per_launch(const Plan& p) { return p.gp ? general_kernels(*p.gp) : 1; }

// alt: for contraction workloads, the general-path view of the same e0; a
// candidate the contraction instantiator cannot map (e.g. a PVU schedule
// that fused loops into floordiv / mod indices) runs through the general
// families (NESTGEN / SIMT-A / GENERIC) instead of being reported
// UNSUPPORTED.
ls_status plan_all(const Workload& w, const GeneralWorkload* gw, const DeviceLimits& lim,
                   const char* const* programs, const size_t* lens, int n, std::vector<Plan>* plans,
                   const GeneralWorkload* alt = nullptr) {
  plans->assign(static_cast<size_t>(n), Plan());
  parallel_for(n, [&](int i) {
    std::string err;
    auto p = parse_program(std::string_view(programs[i], lens[i]), &err);
    Plan& out = (*plans)[static_cast<size_t>(i)];
    if (!p) {
      out.status = P_PARSE;
      out.why = err;
      return;
    }
    if (gw) {
      auto g = std::make_shared<GeneralPlan>(plan_general(*gw, *p, lim));
      out.status = g->status;
      out.why = g->why;
      out.family = g->family;
      std::memcpy(out.cfg, g->cfg, sizeof out.cfg);
      out.gp = g;
      return;
    }
    out = plan_program(w, *p, lim);
    if (out.status == P_UNSUPPORTED && alt) {
      DeviceLimits la = lim;
      la.bf16 = false;  // no tcgen05 conv for a plain contraction
      la.tf32x3 = false;
      auto g = std::make_shared<GeneralPlan>(plan_general(*alt, *p, la));
      if (g->status == P_OK) {
        out = Plan();
        out.status = g->status;
        out.why = g->why;
        out.family = g->family;
        std::memcpy(out.cfg, g->cfg, sizeof out.cfg);
        out.gp = g;
      }
    }
  });
  return LS_OK;
}


// General workload: device buffers for every e0 buffer, reference output by
// the generic executor in fp64 (intermediates in fp64 too).
ls_status set_general_workload(ls_runner* r, const Program& e0, const GeneralWorkload& gw, const std::string& text,
                               const float* const* host_inputs, int n_inputs) {
  int ninp = 0;
  for (int role : gw.roles) ninp += role == 0;
  if (ninp != n_inputs) {
    set_error("ls_runner_set_workload: input count does not match the program's input buffers");
    return LS_ERR_ARG;
  }
  GenProgram gen;
  std::string err;
  if (!encode_generic(e0, &gen, &err)) {
    set_error("e0: " + err);
    return LS_ERR_ARG;
  }
  r->gw = gw;
  r->general = true;
  r->e0_text = text;
  r->w = Workload();
  r->w.c_elems = gw.c_elems;
  const size_t nb = gw.buffers.size();
  r->gbuf.assign(nb, nullptr);
  r->gbuf_dtype.assign(nb, r->bf16 ? 0 : 1);
  std::vector<void*> refbuf(nb, nullptr);
  std::vector<int> refdt(nb, 2);
  const size_t es = r->bf16 ? 2 : 4;
  int inp = 0;
  std::vector<void*> temps;
  for (size_t b = 0; b < nb; ++b) {
    int64_t elems = 1;
    for (int64_t x : gw.shapes[b]) elems *= x;
    const size_t n = static_cast<size_t>(elems);
    if (gw.roles[b] == 0) {  // input: runner dtype, shared by the reference run
      LSB_CUDA(r->pmalloc(&r->gbuf[b], n * es));
      if (r->bf16) {
        float* tmp = nullptr;
        LSB_CUDA(r->pmalloc(reinterpret_cast<void**>(&tmp), n * 4));
        LSB_CUDA(cudaMemcpyAsync(tmp, host_inputs[inp], n * 4, cudaMemcpyHostToDevice, r->st));
        launch_to_bf16(tmp, static_cast<__nv_bfloat16*>(r->gbuf[b]), elems, r->st);
        ++r->setup_launches;
        LSB_CUDA(cudaStreamSynchronize(r->st));
        r->pfree(tmp);
      } else {
        LSB_CUDA(cudaMemcpyAsync(r->gbuf[b], host_inputs[inp], n * 4, cudaMemcpyHostToDevice, r->st));
      }
      ++inp;
      refbuf[b] = r->gbuf[b];
      refdt[b] = r->gbuf_dtype[b];
    } else if (gw.roles[b] == 1 && gw.buffers[b] == gw.c_buf) {  // contraction output
      LSB_CUDA(r->pmalloc(reinterpret_cast<void**>(&r->c), n * 4));
      LSB_CUDA(r->pmalloc(reinterpret_cast<void**>(&r->ref), n * 8));
      r->gbuf[b] = r->c;
      r->gbuf_dtype[b] = 1;
      refbuf[b] = r->ref;
    } else if (gw.roles[b] == 1) {  // the final output of a later stage (e.g. relu)
      LSB_CUDA(r->pmalloc(reinterpret_cast<void**>(&r->c), n * 4));
      LSB_CUDA(r->pmalloc(reinterpret_cast<void**>(&r->ref), n * 8));
      r->gbuf[b] = r->c;
      r->gbuf_dtype[b] = 1;
      r->w.c_elems = elems;
      refbuf[b] = r->ref;
    } else {  // intermediate: fp32 when it holds the contraction's sums, else runner dtype
      if (gw.buffers[b] == gw.c_buf) r->gbuf_dtype[b] = 1;
      LSB_CUDA(r->pmalloc(&r->gbuf[b], n * (r->gbuf_dtype[b] == 1 ? 4 : es)));
      LSB_CUDA(r->pmalloc(&refbuf[b], n * 8));
      temps.push_back(refbuf[b]);
    }
  }
  LSB_CUDA(cudaStreamSynchronize(r->st));  // host inputs consumed; the rest stays queued on r->st
  // reference output: e0 block by block in fp64 (pool blocks are reused in
  // stream order, so the bytecode and fp64 temporaries go back to the pool
  // while the reference run is still queued)
  int64_t* code = nullptr;
  LSB_CUDA(r->pmalloc(reinterpret_cast<void**>(&code), std::max<size_t>(gen.code.size(), 1) * 8));
  LSB_CUDA(cudaMemcpyAsync(code, gen.code.data(), gen.code.size() * 8, cudaMemcpyHostToDevice, r->st));
  GenBuffers B;
  std::memset(&B, 0, sizeof B);
  for (size_t b = 0; b < nb; ++b) {
    B.ptr[b] = refbuf[b];
    B.dtype[b] = refdt[b];
    for (int d = 0; d < gen.ndim[b]; ++d) B.shape[b][d] = gen.shape[b][d];
  }
  for (const GenBlock& g : gen.blocks)
    if (++r->setup_launches, !launch_generic_block(g, code, B, true, nullptr, nullptr, r->st)) {
      set_error("reference run of e0 failed to launch");
      return LS_ERR_CUDA;
    }
  LSB_CUDA(cudaGetLastError());
  r->pfree(code);
  for (void* t : temps) r->pfree(t);
  // K-major weight copy for the tcgen05 conv family: the contraction's
  // weight viewed as [k_rows][n_cols] (n = its contiguous last dim)
  r->tc_ok = false;
  r->lim.bf16 = false;
  r->lim.tf32x3 = false;
  for (size_t b = 0; b < nb; ++b) {
    if (gw.buffers[b] != gw.y_buf || gw.roles[b] != 0) continue;
    const std::vector<int64_t>& sh = gw.shapes[b];
    int64_t elems = 1;
    for (int64_t x : sh) elems *= x;
    r->wt_cols = sh.back();
    r->wt_rows = elems / r->wt_cols;
    if (r->wt_rows % 64 || r->wt_cols % 16) break;
    if (r->bf16) {
      LSB_CUDA(r->pmalloc(&r->wt, static_cast<size_t>(elems) * 2));
      ++r->setup_launches;
      launch_transpose_bf16(static_cast<const __nv_bfloat16*>(r->gbuf[b]), static_cast<__nv_bfloat16*>(r->wt), 1,
                            r->wt_rows, r->wt_cols, r->st);
      LSB_CUDA(cudaGetLastError());
      r->lim.bf16 = true;
    } else {
      // 3xTF32 conv tile: weight halves K-major, and halves of every NHWC
      // input whose channels fill whole 32-element (128-byte) rows
      LSB_CUDA(r->pmalloc(&r->wt, static_cast<size_t>(elems) * 8));
      ++r->setup_launches;
      launch_split_tf32(static_cast<const float*>(r->gbuf[b]), static_cast<float*>(r->wt), 1, r->wt_rows, r->wt_cols,
                        true, r->st);
      r->gbuf_x3.assign(nb, nullptr);
      for (size_t x = 0; x < nb; ++x) {  // inputs split here; intermediates on every launch
        if (gw.roles[x] == 1 || gw.shapes[x].size() != 4 || gw.shapes[x][3] % 32) continue;
        int64_t xe = 1;
        for (int64_t v : gw.shapes[x]) xe *= v;
        LSB_CUDA(r->pmalloc(&r->gbuf_x3[x], static_cast<size_t>(xe) * 8));
        if (gw.roles[x] != 0) continue;
        ++r->setup_launches;
        launch_split_tf32(static_cast<const float*>(r->gbuf[x]), static_cast<float*>(r->gbuf_x3[x]), 1,
                          xe / gw.shapes[x][3], gw.shapes[x][3], false, r->st);
      }
      LSB_CUDA(cudaGetLastError());
      r->lim.tf32x3 = true;
    }
  }
  r->have_workload = true;
  r->best_valid = false;
  return LS_OK;
}

}  // namespace

extern "C" {

ls_status ls_plan_programs(const char* e0, size_t e0_len, const char* const* programs, const size_t* lens, int n,
                           int32_t dtype, ls_result* out) {
  if (!e0 || !out || n < 0 || (n > 0 && (!programs || !lens))) {
    set_error("ls_plan_programs: bad arguments");
    return LS_ERR_ARG;
  }
  std::string err;
  auto p0 = parse_program(std::string_view(e0, e0_len), &err);
  if (!p0) {
    set_error("e0: " + err);
    return LS_ERR_PARSE;
  }
  Workload w;
  GeneralWorkload gw;
  bool general = false;
  if (!analyze_workload(*p0, &w, &err)) {
    std::string err2;
    if (!analyze_general(*p0, &gw, &err2)) {
      set_error("e0: " + err + "; " + err2);
      return LS_ERR_ARG;
    }
    general = true;
  }
  DeviceLimits lim;
  lim.bf16 = !general && dtype == LS_DTYPE_BF16 && w.x_kmajor && w.sc[R_N] == 1;
  lim.tf32x3 = !general && dtype != LS_DTYPE_BF16 && w.x_kmajor && w.sc[R_N] == 1;
  if (general)
    for (size_t b = 0; b < gw.buffers.size(); ++b)
      if (gw.buffers[b] == gw.y_buf && gw.roles[b] == 0) {
        int64_t elems = 1;
        for (int64_t x : gw.shapes[b]) elems *= x;
        const bool ok = (elems / gw.shapes[b].back()) % 64 == 0 && gw.shapes[b].back() % 16 == 0;
        (dtype == LS_DTYPE_BF16 ? lim.bf16 : lim.tf32x3) = ok;
      }
  std::vector<Plan> plans;
  GeneralWorkload alt;
  std::string aerr;
  const bool has_alt = !general && analyze_general(*p0, &alt, &aerr);
  plan_all(w, general ? &gw : nullptr, lim, programs, lens, n, &plans, has_alt ? &alt : nullptr);
  for (int i = 0; i < n; ++i) fill_result(plans[static_cast<size_t>(i)], &out[i]);
  return LS_OK;
}

ls_status ls_runner_create(int device, const ls_runner_opts* opts, ls_runner** out) {
  if (!out) {
    set_error("ls_runner_create: null out");
    return LS_ERR_ARG;
  }
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
    cudaGetLastError();
    set_error("no CUDA device: the B200 runner has no CPU fallback");
    return LS_ERR_CUDA;
  }
  if (device < 0 || device >= count) {
    set_error("device index out of range");
    return LS_ERR_ARG;
  }
  LSB_CUDA(cudaSetDevice(device));
  cudaDeviceProp prop;
  LSB_CUDA(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10) {
    set_error("the runner's kernels are compiled for sm_100a (B200)");
    return LS_ERR_CUDA;
  }
  auto r = std::make_unique<ls_runner>();
  r->device = device;
  ls_runner_opts o{};
  o.dtype = LS_DTYPE_BF16;
  o.min_repeats = 3;
  o.max_repeats = 200;
  o.target_ms = 0.2;
  o.timeout_ms = 2.0;
  o.rtol = 0.0;
  o.atol = 0.0;
  o.timeout_factor = 0.0;
  o.timeout_floor_ms = 0.05;
  o.single_shot_factor = 0.0;
  if (opts) o = *opts;
  if (o.min_repeats < 1) o.min_repeats = 1;
  if (o.max_repeats < o.min_repeats) o.max_repeats = o.min_repeats;
  r->opts = o;
  r->bf16 = o.dtype == LS_DTYPE_BF16;
  r->lim.max_threads = prop.maxThreadsPerBlock;
  r->lim.max_smem = static_cast<int64_t>(prop.sharedMemPerBlockOptin) - 1024;
  LSB_CUDA(cudaStreamCreateWithFlags(&r->st, cudaStreamNonBlocking));
  LSB_CUDA(cudaStreamCreateWithFlags(&r->cap_st, cudaStreamNonBlocking));
  LSB_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&r->gate), 64, cudaHostAllocMapped | cudaHostAllocPortable));
  *r->gate = 0;
  {  // every runner kernel loaded now, not lazily inside a timed checked launch
    static std::once_flag once;
    std::call_once(once, [] {
      preload_simt_kernels();
      preload_simta_f32();
      preload_simta_bf16();
      preload_tc_gemm();
      preload_tc_conv();
      preload_generic_kernels();
    });
  }
  LSB_CUDA(cudaMalloc(&r->deadline, 8 * sizeof(unsigned long long)));
  ls_status s = r->ensure_capacity(256);
  if (s != LS_OK) return s;
  // calibrate the device-side elapsed time of an empty candidate (arm kernel,
  // event, one empty kernel launch, event, stamp kernel: the launch gaps a real
  // candidate's elapsed time also carries), so the best-so-far behind every
  // deadline is the kernel time
  {
    unsigned long long init[8] = {0, 0, ~0ull, 0, 0, 0, 0, 0};
    LSB_CUDA(cudaMemcpy(r->deadline, init, sizeof init, cudaMemcpyHostToDevice));
    cudaEvent_t e;
    LSB_CUDA(cudaEventCreate(&e));
    unsigned long long best = ~0ull;
    for (int i = 0; i < 16; ++i) {
      launch_gate(r->gate, ++r->gate_seq, kGateMaxNs, r->st);
      launch_arm(r->deadline, nullptr, nullptr, 0.0, 0, 0, r->st);
      LSB_CUDA(cudaEventRecord(e, r->st));
      launch_delay(0, r->st);  // stands in for the candidate's own launch
      LSB_CUDA(cudaEventRecord(e, r->st));
      launch_stamp(r->deadline, r->st);
      r->open_gate(r->gate_seq);
      unsigned long long h[4];
      LSB_CUDA(cudaMemcpyAsync(h, r->deadline, sizeof h, cudaMemcpyDeviceToHost, r->st));
      LSB_CUDA(cudaStreamSynchronize(r->st));
      if (h[3] > h[1]) best = std::min(best, h[3] - h[1]);
    }
    cudaEventDestroy(e);
    r->empty_ns = best == ~0ull ? 0 : best;
  }
  *out = r.release();
  return LS_OK;
}

ls_status ls_runner_set_workload(ls_runner* r, const char* e0, size_t len, const float* const* host_inputs,
                                 int n_inputs) {
  if (!r || !e0 || !host_inputs) {
    set_error("ls_runner_set_workload: bad arguments");
    return LS_ERR_ARG;
  }
  LSB_CUDA(cudaSetDevice(r->device));
  LSB_CUDA(cudaStreamSynchronize(r->st));
  r->release_workload();
  std::string err;
  auto p0 = parse_program(std::string_view(e0, len), &err);
  if (!p0) {
    set_error("e0: " + err);
    return LS_ERR_PARSE;
  }
  Workload w;
  if (!analyze_workload(*p0, &w, &err)) {
    GeneralWorkload gw;
    std::string err2;
    if (!analyze_general(*p0, &gw, &err2)) {
      set_error("e0: " + err + "; " + err2);
      return LS_ERR_ARG;
    }
    return set_general_workload(r, *p0, gw, std::string(e0, len), host_inputs, n_inputs);
  }
  if (static_cast<int>(w.input_bufs.size()) != n_inputs) {
    set_error("ls_runner_set_workload: input count does not match the program's input buffers");
    return LS_ERR_ARG;
  }
  r->w = w;
  r->e0_text.assign(e0, len);
  for (int i = 0; i < 4; ++i) {
    r->s.sx[i] = w.sx[i];
    r->s.sy[i] = w.sy[i];
    r->s.sc[i] = w.sc[i];
    r->s.ext[i] = w.extent[i];
  }
  const size_t es = r->bf16 ? 2 : 4;
  auto upload = [&](int buf, int64_t elems, void** dst) -> ls_status {
    int idx = -1;
    for (int i = 0; i < n_inputs; ++i)
      if (w.input_bufs[static_cast<size_t>(i)] == buf) idx = i;
    if (idx < 0) {
      set_error("operand is not an input buffer");
      return LS_ERR_ARG;
    }
    LSB_CUDA(r->pmalloc(dst, static_cast<size_t>(elems) * es));
    if (!r->bf16) {
      LSB_CUDA(cudaMemcpyAsync(*dst, host_inputs[idx], static_cast<size_t>(elems) * 4, cudaMemcpyHostToDevice, r->st));
    } else {
      float* tmp = nullptr;
      LSB_CUDA(r->pmalloc(reinterpret_cast<void**>(&tmp), static_cast<size_t>(elems) * 4));
      LSB_CUDA(cudaMemcpyAsync(tmp, host_inputs[idx], static_cast<size_t>(elems) * 4, cudaMemcpyHostToDevice, r->st));
      launch_to_bf16(tmp, static_cast<__nv_bfloat16*>(*dst), elems, r->st);
      ++r->setup_launches;
      LSB_CUDA(cudaStreamSynchronize(r->st));
      r->pfree(tmp);
    }
    return LS_OK;
  };
  ls_status s;
  if ((s = upload(w.x_buf, w.x_elems, &r->x)) != LS_OK) return s;
  if ((s = upload(w.y_buf, w.y_elems, &r->y)) != LS_OK) return s;
  // the host inputs are consumed once the uploads are done; the reference
  // run and the operand copies below stay queued on r->st, so the first
  // measure call plans its batch on the host while they run
  LSB_CUDA(cudaStreamSynchronize(r->st));
  LSB_CUDA(r->pmalloc(reinterpret_cast<void**>(&r->c), static_cast<size_t>(w.c_elems) * 4));
  LSB_CUDA(r->pmalloc(reinterpret_cast<void**>(&r->ref), static_cast<size_t>(w.c_elems) * 8));
  launch_reference(r->x, r->y, r->ref, r->s, r->bf16, r->st);
  ++r->setup_launches;
  LSB_CUDA(cudaGetLastError());

  // tcgen05 operands: X must be [batch][M][K]; Y is used K-major ([batch][N][K]),
  // transposed once here when the workload stores it [batch][K][N].  fp32
  // workloads get both as [hi | lo] halves for the 3xTF32 tile.
  const int64_t B = w.extent[R_BATCH], M = w.extent[R_M], N = w.extent[R_N], K = w.extent[R_K];
  bool x_ok = w.x_kmajor && w.sx[R_M] == K && (!w.has_batch || w.sx[R_BATCH] == M * K);
  bool y_kmaj = w.y_kmajor && w.sy[R_N] == K && (!w.has_batch || w.sy[R_BATCH] == N * K);
  bool y_nmaj = !w.y_kmajor && w.sy[R_N] == 1 && w.sy[R_K] == N && (!w.has_batch || w.sy[R_BATCH] == N * K);
  bool c_ok = w.sc[R_N] == 1 && w.sc[R_M] == N && (!w.has_batch || w.sc[R_BATCH] == M * N);
  r->tc_ok = x_ok && (y_kmaj || y_nmaj) && c_ok && K % 64 == 0 && M % 128 == 0;
  if (r->tc_ok && !r->bf16) {
    LSB_CUDA(r->pmalloc(&r->xs, static_cast<size_t>(w.x_elems) * 8));
    LSB_CUDA(r->pmalloc(&r->yk, static_cast<size_t>(w.y_elems) * 8));
    launch_split_tf32(static_cast<const float*>(r->x), static_cast<float*>(r->xs), B, M, K, false, r->st);
    r->setup_launches += 2;
    if (y_kmaj) launch_split_tf32(static_cast<const float*>(r->y), static_cast<float*>(r->yk), B, N, K, false, r->st);
    else launch_split_tf32(static_cast<const float*>(r->y), static_cast<float*>(r->yk), B, K, N, true, r->st);
    LSB_CUDA(cudaGetLastError());
    if (!make_kmajor_map(&r->tmap_a, r->xs, 2 * B, M, K, 128, true)) {
      set_error("cuTensorMapEncodeTiled failed for the A operand halves");
      return LS_ERR_CUDA;
    }
    r->have_tmap_c = make_c_map(&r->tmap_c, r->c, B, M, N);
  } else if (r->tc_ok) {
    if (y_kmaj) {
      r->yk = nullptr;
      LSB_CUDA(r->pmalloc(&r->yk, static_cast<size_t>(w.y_elems) * 2));
      LSB_CUDA(cudaMemcpyAsync(r->yk, r->y, static_cast<size_t>(w.y_elems) * 2, cudaMemcpyDeviceToDevice, r->st));
    } else {
      LSB_CUDA(r->pmalloc(&r->yk, static_cast<size_t>(w.y_elems) * 2));
      ++r->setup_launches;
      launch_transpose_bf16(static_cast<const __nv_bfloat16*>(r->y), static_cast<__nv_bfloat16*>(r->yk), B, K, N,
                            r->st);
      LSB_CUDA(cudaGetLastError());
    }
    if (!make_kmajor_map(&r->tmap_a, r->x, B, M, K, 128)) {
      set_error("cuTensorMapEncodeTiled failed for the A operand");
      return LS_ERR_CUDA;
    }
    r->have_tmap_c = make_c_map(&r->tmap_c, r->c, B, M, N);
  }
  r->lim.bf16 = r->tc_ok && r->bf16;
  r->lim.tf32x3 = r->tc_ok && !r->bf16;
  {  // general-path view of the same buffers for candidates plan_program cannot map
    GeneralWorkload alt;
    std::string aerr;
    if (analyze_general(*p0, &alt, &aerr) && alt.buffers.size() == 3) {
      const std::string xn = p0->buffers[static_cast<size_t>(w.x_buf)].name;
      const std::string yn = p0->buffers[static_cast<size_t>(w.y_buf)].name;
      const std::string cn = p0->buffers[static_cast<size_t>(w.c_buf)].name;
      r->gbuf.assign(3, nullptr);
      r->gbuf_dtype.assign(3, 1);
      bool ok = true;
      for (size_t b = 0; b < 3; ++b) {
        const std::string& nm = alt.buffers[b];
        if (nm == xn) { r->gbuf[b] = r->x; r->gbuf_dtype[b] = r->bf16 ? 0 : 1; }
        else if (nm == yn) { r->gbuf[b] = r->y; r->gbuf_dtype[b] = r->bf16 ? 0 : 1; }
        else if (nm == cn) { r->gbuf[b] = r->c; r->gbuf_dtype[b] = 1; }
        else ok = false;
      }
      if (ok) {
        r->gw = alt;
        r->has_alt = true;
      } else {
        r->gbuf.clear();
        r->gbuf_dtype.clear();
      }
    }
  }
  r->have_workload = true;
  r->best_valid = false;
  return LS_OK;
}

ls_status ls_runner_plan(ls_runner* r, const char* const* programs, const size_t* lens, int n, ls_result* out) {
  if (!r || !r->have_workload) {
    set_error("ls_runner_plan: no workload");
    return LS_ERR_STATE;
  }
  std::vector<Plan> plans;
  const auto tp0 = std::chrono::steady_clock::now();
  plan_all(r->w, r->general ? &r->gw : nullptr, r->lim, programs, lens, n, &plans,
           r->has_alt ? &r->gw : nullptr);
  const double plan_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tp0).count();
  for (int i = 0; i < n; ++i) fill_result(plans[static_cast<size_t>(i)], &out[i]);
  return LS_OK;
}

ls_status ls_runner_measure(ls_runner* r, const char* const* programs, const size_t* lens, int n, ls_result* out) {
  if (!r || !out || n < 0 || (n > 0 && (!programs || !lens))) {
    set_error("ls_runner_measure: bad arguments");
    return LS_ERR_ARG;
  }
  if (!r->have_workload) {
    set_error("ls_runner_measure: set a workload first");
    return LS_ERR_STATE;
  }
  LSB_CUDA(cudaSetDevice(r->device));
  ls_status s = r->ensure_capacity(n);
  if (s != LS_OK) return s;
  std::vector<Plan> plans;
  const auto tp0 = std::chrono::steady_clock::now();
  plan_all(r->w, r->general ? &r->gw : nullptr, r->lim, programs, lens, n, &plans,
           r->has_alt ? &r->gw : nullptr);
  const double plan_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tp0).count();
  for (int i = 0; i < n; ++i) fill_result(plans[static_cast<size_t>(i)], &out[i]);
  r->launches = r->setup_launches;  // the preceding set_workload's kernels are counted once, here
  r->setup_launches = 0;
  bool any_gp = false;
  for (const Plan& p : plans) any_gp |= p.gp != nullptr;
  if (any_gp) {  // one upload of every candidate's bytecode
    std::vector<int64_t> all;
    std::vector<size_t> at(static_cast<size_t>(n), 0);
    for (int i = 0; i < n; ++i) {
      const Plan& p = plans[static_cast<size_t>(i)];
      if (p.status != P_OK || !p.gp) continue;
      at[static_cast<size_t>(i)] = all.size();
      all.insert(all.end(), p.gp->gen.code.begin(), p.gp->gen.code.end());
    }
    if (all.size() > r->gcode_cap) {
      cudaFree(r->gcode);
      r->gcode = nullptr;
      r->gcode_cap = std::max(all.size(), 2 * r->gcode_cap);
      LSB_CUDA(cudaMalloc(&r->gcode, r->gcode_cap * 8));
    }
    if (!all.empty()) LSB_CUDA(cudaMemcpyAsync(r->gcode, all.data(), all.size() * 8, cudaMemcpyHostToDevice, r->st));
    for (int i = 0; i < n; ++i)
      if (plans[static_cast<size_t>(i)].gp) plans[static_cast<size_t>(i)].gcode = r->gcode + at[static_cast<size_t>(i)];
  }
  const size_t cbytes = static_cast<size_t>(r->w.c_elems) * sizeof(float);
  const unsigned long long timeout_ns = static_cast<unsigned long long>(r->opts.timeout_ms * 1e6);
  LSB_CUDA(cudaMemsetAsync(r->flags, 0, static_cast<size_t>(n) * sizeof(int), r->st));
  LSB_CUDA(cudaMemsetAsync(r->parity, 0, static_cast<size_t>(n) * 16, r->st));
  s = r->prepare_sync(plans);
  if (s != LS_OK) return s;
  cudaEvent_t* E = r->ev.data();
  cudaEvent_t batch0;
  LSB_CUDA(cudaEventCreate(&batch0));
  LSB_CUDA(cudaEventRecord(batch0, r->st));

  auto host_now = [] { return std::chrono::duration<double, std::milli>(
                            std::chrono::steady_clock::now().time_since_epoch()).count(); };
  std::memset(r->stats, 0, sizeof r->stats);
  r->stats[3] = plan_ms;
  r->stats[4] = static_cast<double>(r->empty_ns) / 1e3;
  double h0 = host_now();
  // ---- phase A: checked run ----
  // C starts poisoned (NaN) and the parity reducer re-poisons it, so any
  // element a candidate fails to write is a mismatch.  The deadline of each
  // checked launch is armed on the device from the best time seen so far.
  std::vector<char> launched(static_cast<size_t>(n), 0);
  const unsigned long long best_init[5] = {0, 0, ~0ull, 0, r->empty_ns};
  if (!r->opts.carry_best || !r->best_valid) {
    LSB_CUDA(cudaMemcpyAsync(r->deadline, best_init, sizeof best_init, cudaMemcpyHostToDevice, r->st));
    r->best_valid = true;
  }
  LSB_CUDA(cudaMemsetAsync(r->c, 0xFF, cbytes, r->st));
  const unsigned long long floor_ns = static_cast<unsigned long long>(r->opts.timeout_floor_ms * 1e6);
  // checked-run order: families expected to be fast first, so the device-side
  // best-so-far (and with it every later deadline) drops early; results are
  // still reported in candidate order
  std::vector<int> order;
  {
    auto rank = [](int fam) {
      switch (fam) {
        case F_TC: case F_TCCONV: return 0;
        case F_SIMT: case F_SIMTA: return 1;
        case F_NAIVE: case F_GENERIC: return 2;
        default: return 3;  // LOOPNEST, NESTGEN
      }
    };
    for (int pass = 0; pass < 4; ++pass)
      for (int i = 0; i < n; ++i)
        if (plans[static_cast<size_t>(i)].status == P_OK && rank(plans[static_cast<size_t>(i)].family) == pass)
          order.push_back(i);
  }
  // phase-B graphs of fast candidates are captured on a helper thread while
  // the device is still running phase A: a candidate's repeat count depends
  // only on its own checked-launch time, known once its E1 event completes.
  // The capture stream never executes; graphs are launched on r->st in
  // phase B (a graph that ends up unused -- timeout, single-shot -- is
  // destroyed).
  auto reps_for = [&](float warm_ms) {
    double wm = std::max(1e-4, static_cast<double>(warm_ms));
    int rep = static_cast<int>(std::ceil(r->opts.target_ms / wm));
    return std::max(r->opts.min_repeats, std::min(r->opts.max_repeats, rep));
  };
  auto graph_eligible = [&](float warm_ms) {
    return r->opts.flush_l2 == 0 && std::max(1e-4, static_cast<double>(warm_ms)) < 0.02;
  };
  std::vector<cudaGraphExec_t> pre_exec(static_cast<size_t>(n), nullptr);
  std::vector<int> pre_rep(static_cast<size_t>(n), 0);
  std::vector<char> enq_ok(static_cast<size_t>(n), 0);
  std::atomic<int> enq_done{0};
  std::atomic<bool> enq_stop{false};
  std::thread helper;
  if (r->opts.flush_l2 == 0 && !order.empty()) {
    helper = std::thread([&] {
      cudaSetDevice(r->device);
      // start only once the enqueue loop is done: capturing beside it slows
      // the main thread's launches (driver lock), and host gaps between an
      // arm kernel and its candidate would inflate the checked-launch times
      const int total = static_cast<int>(order.size());
      while (enq_done.load(std::memory_order_acquire) < total && !enq_stop.load(std::memory_order_acquire))
        std::this_thread::sleep_for(std::chrono::microseconds(50));
      for (int k = 0; k < total; ++k) {
        while (enq_done.load(std::memory_order_acquire) <= k) {
          if (enq_stop.load(std::memory_order_acquire) && enq_done.load(std::memory_order_acquire) <= k) return;
          std::this_thread::yield();
        }
        const int i = order[static_cast<size_t>(k)];
        if (!enq_ok[static_cast<size_t>(i)]) continue;
        if (cudaEventSynchronize(E[4 * i + 1]) != cudaSuccess) return;
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, E[4 * i], E[4 * i + 1]) != cudaSuccess || !graph_eligible(ms)) continue;
        const int rep = reps_for(ms);
        const Plan& p = plans[static_cast<size_t>(i)];
        cudaGraph_t g = nullptr;
        cudaGraphExec_t ge = nullptr;
        bool ok = cudaStreamBeginCapture(r->cap_st, cudaStreamCaptureModeThreadLocal) == cudaSuccess;
        for (int k2 = 0; ok && k2 < rep; ++k2) ok = r->launch(p, false, i, r->cap_st);
        cudaError_t ce = cudaStreamEndCapture(r->cap_st, &g);
        ok = ok && ce == cudaSuccess && g && cudaGraphInstantiate(&ge, g, 0) == cudaSuccess;
        if (g) cudaGraphDestroy(g);
        if (!ok) {
          cudaGetLastError();
          if (ge) cudaGraphExecDestroy(ge);
          r->launches -= kernels_per_launch(p) * rep;  // counted by launch(), never run
          continue;
        }
        pre_exec[static_cast<size_t>(i)] = ge;
        pre_rep[static_cast<size_t>(i)] = rep;
      }
    });
  }
  struct HelperJoin {  // also on an early error return out of the enqueue loop
    std::thread& t;
    std::atomic<bool>& stop;
    void operator()() {
      if (!t.joinable()) return;
      stop.store(true, std::memory_order_release);
      t.join();
    }
    ~HelperJoin() { (*this)(); }
  } join_helper{helper, enq_stop};
  // checked launches are enqueued in gated chunks: the device starts a chunk
  // only once the host has enqueued all of it
  unsigned int seq = r->gate_seq;
  int in_chunk = 0;
  int prev = -1;
  for (int i : order) {
    const Plan& p = plans[static_cast<size_t>(i)];
    if (in_chunk == 0) {
      launch_gate(r->gate, ++seq, kGateMaxNs, r->st);
      ++r->launches;
      r->gate_seq = seq;
    }
    if (++in_chunk == kGateChunk) in_chunk = 0;
    struct ChunkEnd {  // opens the chunk's gate once its last candidate is enqueued (or on any exit)
      ls_runner* r;
      unsigned int seq;
      bool last;
      ~ChunkEnd() { if (last) r->open_gate(seq); }
    } chunk_end{r, seq, in_chunk == 0};
    launch_arm(r->deadline, prev >= 0 ? r->flags + prev : nullptr, prev >= 0 ? r->parity + 2 * prev : nullptr,
               r->opts.timeout_factor, floor_ns, timeout_ns, r->st);
    ++r->launches;
    LSB_CUDA(cudaEventRecord(E[4 * i], r->st));
    bool ok = r->launch(p, true, i);
    LSB_CUDA(cudaEventRecord(E[4 * i + 1], r->st));
    launch_stamp(r->deadline, r->st);
    ++r->launches;
    if (!ok) {
      cudaGetLastError();
      out[i].status = LS_RUN_LAUNCH;
      enq_done.fetch_add(1, std::memory_order_release);
      // the next arm kernel must not take this empty slot's arm-to-stamp gap
      // as a candidate time (the last good candidate was already accounted
      // for by this slot's own arm kernel)
      prev = -1;
      cudaError_t me = cudaMemsetAsync(r->c, 0xFF, cbytes, r->st);
      if (me != cudaSuccess) {
        join_helper();
        LSB_CUDA(me);
      }
      continue;
    }
    launch_parity(r->c, r->ref, r->w.c_elems, r->opts.rtol, r->opts.atol, r->parity + 2 * i, true, r->st);
    ++r->launches;
    launched[static_cast<size_t>(i)] = 1;
    enq_ok[static_cast<size_t>(i)] = 1;
    enq_done.fetch_add(1, std::memory_order_release);
    prev = i;
  }
  r->open_gate(seq);
  r->stats[6] = host_now() - h0;  // phase A enqueue only (before waiting for the device)
  enq_stop.store(true, std::memory_order_release);  // enqueue finished (or aborted): the helper may start
  cudaError_t se = cudaStreamSynchronize(r->st);
  join_helper();
  // an unused pre-captured graph: destroyed, its kernels uncounted
  auto drop_one = [&](int i) {
    cudaGraphExec_t& g = pre_exec[static_cast<size_t>(i)];
    if (!g) return;
    cudaGraphExecDestroy(g);
    g = nullptr;
    r->launches -= kernels_per_launch(plans[static_cast<size_t>(i)]) * pre_rep[static_cast<size_t>(i)];
  };
  auto drop_pre = [&] {
    for (int i = 0; i < n; ++i) drop_one(i);
  };
  if (se != cudaSuccess) {
    drop_pre();
    cudaEventDestroy(batch0);
    set_error(std::string("runner phase A: ") + cudaGetErrorString(se));
    return LS_ERR_CUDA;
  }
  for (int i = 0; i < n; ++i)
    if (out[i].status == LS_RUN_OK && !launched[static_cast<size_t>(i)]) out[i].status = LS_RUN_LAUNCH;
  {  // diagnostics: the device-side best-so-far after phase A (debug_stats[5], us)
    unsigned long long dev_state[5];
    if (cudaMemcpy(dev_state, r->deadline, sizeof dev_state, cudaMemcpyDeviceToHost) == cudaSuccess)
      r->stats[5] = dev_state[2] == ~0ull ? -1.0 : static_cast<double>(dev_state[2]) / 1e3;
  }
  std::vector<int> tflag(static_cast<size_t>(n));
  std::vector<unsigned long long> par(static_cast<size_t>(2 * n));
  LSB_CUDA(cudaMemcpy(tflag.data(), r->flags, static_cast<size_t>(n) * sizeof(int), cudaMemcpyDeviceToHost));
  LSB_CUDA(cudaMemcpy(par.data(), r->parity, static_cast<size_t>(n) * 16, cudaMemcpyDeviceToHost));
  std::vector<float> warm(static_cast<size_t>(n), 0.f);
  for (int i = 0; i < n; ++i) {
    if (!launched[static_cast<size_t>(i)]) continue;
    LSB_CUDA(cudaEventElapsedTime(&warm[static_cast<size_t>(i)], E[4 * i], E[4 * i + 1]));
    out[i].checked_ns = 1e6 * static_cast<double>(warm[static_cast<size_t>(i)]);
    double err;
    unsigned long long bits = par[static_cast<size_t>(2 * i)];
    std::memcpy(&err, &bits, sizeof err);
    out[i].max_abs_err = err;
    out[i].mismatches = static_cast<int64_t>(par[static_cast<size_t>(2 * i + 1)]);
    if (tflag[static_cast<size_t>(i)]) {
      out[i].status = LS_RUN_TIMEOUT;
      out[i].latency_ns = 1e6 * static_cast<double>(warm[static_cast<size_t>(i)]);  // abort time: lower bound
      out[i].repeats = 1;
      launched[static_cast<size_t>(i)] = 0;
    } else if (out[i].mismatches) {
      out[i].status = LS_RUN_PARITY;  // no timed repeats: latency is the checked launch
      out[i].latency_ns = 1e6 * static_cast<double>(warm[static_cast<size_t>(i)]);
      out[i].repeats = 0;
      launched[static_cast<size_t>(i)] = 0;
    }
  }

  r->stats[0] = host_now() - h0;
  h0 = host_now();
  // ---- phase B: timed repeats ----
  // Each candidate's repeats are captured into one CUDA graph (PDL edges
  // between tcgen05 launches are preserved) and the graph launch is
  // bracketed by two events, so no host launch gap can enter the timing.
  // If capture fails the repeats are launched directly behind a device spin
  // sized to the host enqueue time.
  std::vector<int> reps(static_cast<size_t>(n), 0);
  // slow candidates (checked launch > single_shot_factor x the fastest one)
  // are not worth timed repeats: they report their checked launch
  std::vector<char> single(static_cast<size_t>(n), 0);
  if (r->opts.single_shot_factor > 0.0) {
    float best_warm = 0.f;
    for (int i = 0; i < n; ++i)
      if (launched[static_cast<size_t>(i)] && out[i].status == LS_RUN_OK &&
          (best_warm == 0.f || warm[static_cast<size_t>(i)] < best_warm))
        best_warm = warm[static_cast<size_t>(i)];
    for (int i = 0; i < n; ++i)
      if (launched[static_cast<size_t>(i)] && best_warm > 0.f &&
          warm[static_cast<size_t>(i)] > r->opts.single_shot_factor * best_warm) {
        single[static_cast<size_t>(i)] = 1;
        launched[static_cast<size_t>(i)] = 0;
        out[i].repeats = 0;
        out[i].latency_ns = 1e6 * static_cast<double>(warm[static_cast<size_t>(i)]);
      }
  }
  std::vector<cudaGraphExec_t> execs;
  struct ColdEv {
    int i;
    cudaEvent_t a, b;
  };
  std::vector<ColdEv> cold_ev;  // flush_l2: one event pair per timed repeat
  struct ColdEvFree {
    std::vector<ColdEv>& v;
    ~ColdEvFree() {
      for (const ColdEv& c : v) {
        cudaEventDestroy(c.a);
        cudaEventDestroy(c.b);
      }
    }
  } cold_free{cold_ev};
  const int chunk = 32;
  double prev_gpu_us = 0.0;
  for (int c0 = 0; c0 < n; c0 += chunk) {
    int c1 = std::min(n, c0 + chunk);
    std::vector<cudaGraphExec_t> ge(static_cast<size_t>(c1 - c0), nullptr);
    int64_t direct_calls = 0;
    double gpu_us = 0.0;
    for (int i = c0; i < c1; ++i) {
      if (!launched[static_cast<size_t>(i)]) continue;
      const Plan& p = plans[static_cast<size_t>(i)];
      double wm = std::max(1e-4, static_cast<double>(warm[static_cast<size_t>(i)]));
      const int rep = reps_for(warm[static_cast<size_t>(i)]);
      reps[static_cast<size_t>(i)] = rep;
      gpu_us += rep * wm * 1e3;
      if (pre_exec[static_cast<size_t>(i)] && pre_rep[static_cast<size_t>(i)] == rep) {
        ge[static_cast<size_t>(i - c0)] = pre_exec[static_cast<size_t>(i)];  // captured during phase A
        pre_exec[static_cast<size_t>(i)] = nullptr;
      } else if (graph_eligible(warm[static_cast<size_t>(i)])) {
        // graphs only where launch gaps could matter: fast candidates (the
        // instantiation costs ~0.05 ms of host time per candidate)
        drop_one(i);
        cudaGraph_t g = nullptr;
        bool ok = cudaStreamBeginCapture(r->st, cudaStreamCaptureModeThreadLocal) == cudaSuccess;
        for (int k = 0; ok && k < rep; ++k) ok = r->launch(p, false, i);
        cudaError_t ce = cudaStreamEndCapture(r->st, &g);
        ok = ok && ce == cudaSuccess && g &&
             cudaGraphInstantiate(&ge[static_cast<size_t>(i - c0)], g, 0) == cudaSuccess;
        if (g) cudaGraphDestroy(g);
        if (!ok) {
          cudaGetLastError();
          ge[static_cast<size_t>(i - c0)] = nullptr;
        }
      }
      if (!ge[static_cast<size_t>(i - c0)]) direct_calls += rep * (p.needs_zero ? 2 : 1) + 2;
    }
    if (direct_calls) {
      double spin = r->launch_host_us * static_cast<double>(direct_calls) - prev_gpu_us;
      if (spin > 0) {
        r->stats[2] += std::min(spin, 20000.0);
        launch_delay(static_cast<unsigned long long>(std::min(spin, 20000.0) * 1e3), r->st);
        ++r->launches;
      }
    }
    for (int i = c0; i < c1; ++i) {
      if (!launched[static_cast<size_t>(i)]) continue;
      const Plan& p = plans[static_cast<size_t>(i)];
      cudaGraphExec_t g = ge[static_cast<size_t>(i - c0)];
      // the graph's device-side upload (otherwise done by its first launch,
      // inside the timed region) precedes the start event
      if (g) LSB_CUDA(cudaGraphUpload(g, r->st));
      if (r->opts.flush_l2) {
        // cold-L2 latency: every repeat runs after a 256 MB scrub and is
        // timed alone (events around the candidate's launch only)
        if (!r->scrub) LSB_CUDA(cudaMalloc(&r->scrub, ls_runner::kScrubBytes));
        const int rep = reps[static_cast<size_t>(i)];
        for (int k = 0; k < rep; ++k) {
          cudaEvent_t a, b;
          LSB_CUDA(cudaEventCreate(&a));
          LSB_CUDA(cudaEventCreate(&b));
          cold_ev.push_back({i, a, b});
          LSB_CUDA(cudaMemsetAsync(r->scrub, k & 0xff, ls_runner::kScrubBytes, r->st));
          LSB_CUDA(cudaEventRecord(a, r->st));
          if (!r->launch(p, false, i)) {
            set_error("runner phase B: launch failed");
            cudaEventDestroy(batch0);
            return LS_ERR_CUDA;
          }
          LSB_CUDA(cudaEventRecord(b, r->st));
        }
        continue;
      }
      LSB_CUDA(cudaEventRecord(E[4 * i + 2], r->st));
      if (g) {
        LSB_CUDA(cudaGraphLaunch(g, r->st));
        execs.push_back(g);
      } else {
        for (int k = 0; k < reps[static_cast<size_t>(i)]; ++k)
          if (!r->launch(p, false, i)) {
            set_error("runner phase B: launch failed");
            cudaEventDestroy(batch0);
            return LS_ERR_CUDA;
          }
      }
      LSB_CUDA(cudaEventRecord(E[4 * i + 3], r->st));
    }
    prev_gpu_us = gpu_us;
  }
  drop_pre();  // timed out / single-shot / parity-failed before phase B
  r->stats[1] = host_now() - h0;
  cudaEvent_t batch1;
  LSB_CUDA(cudaEventCreate(&batch1));
  LSB_CUDA(cudaEventRecord(batch1, r->st));
  se = cudaStreamSynchronize(r->st);
  for (cudaGraphExec_t g : execs) cudaGraphExecDestroy(g);
  if (se != cudaSuccess) {
    set_error(std::string("runner phase B: ") + cudaGetErrorString(se));
    return LS_ERR_CUDA;
  }
  std::vector<double> cold_ms(static_cast<size_t>(n), 0.0);
  for (const ColdEv& c : cold_ev) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, c.a, c.b) == cudaSuccess) cold_ms[static_cast<size_t>(c.i)] += ms;
  }
  for (int i = 0; i < n; ++i) {
    if (!launched[static_cast<size_t>(i)]) continue;
    float ms = 0.f;
    if (r->opts.flush_l2) ms = static_cast<float>(cold_ms[static_cast<size_t>(i)]);
    else LSB_CUDA(cudaEventElapsedTime(&ms, E[4 * i + 2], E[4 * i + 3]));
    out[i].repeats = reps[static_cast<size_t>(i)];
    out[i].latency_ns = 1e6 * static_cast<double>(ms) / reps[static_cast<size_t>(i)];
  }
  cudaEventElapsedTime(&r->last_ms, batch0, batch1);
  cudaEventDestroy(batch0);
  cudaEventDestroy(batch1);
  return LS_OK;
}

ls_status ls_runner_baseline(ls_runner* r, ls_result* out) {
  if (!r || !r->have_workload) {
    set_error("ls_runner_baseline: no workload");
    return LS_ERR_STATE;
  }
  const char* t = r->e0_text.c_str();
  size_t l = r->e0_text.size();
  return ls_runner_measure(r, &t, &l, 1, out);
}

ls_status ls_runner_last_output(ls_runner* r, float* host, size_t count) {
  if (!r || !r->have_workload || !host || count > static_cast<size_t>(r->w.c_elems)) {
    set_error("ls_runner_last_output: bad arguments");
    return LS_ERR_ARG;
  }
  LSB_CUDA(cudaSetDevice(r->device));
  LSB_CUDA(cudaStreamSynchronize(r->st));
  LSB_CUDA(cudaMemcpy(host, r->c, count * 4, cudaMemcpyDeviceToHost));
  return LS_OK;
}

ls_status ls_runner_reference_output(ls_runner* r, double* host, size_t count) {
  if (!r || !r->have_workload || !host || count > static_cast<size_t>(r->w.c_elems)) {
    set_error("ls_runner_reference_output: bad arguments");
    return LS_ERR_ARG;
  }
  LSB_CUDA(cudaSetDevice(r->device));
  LSB_CUDA(cudaStreamSynchronize(r->st));
  LSB_CUDA(cudaMemcpy(host, r->ref, count * 8, cudaMemcpyDeviceToHost));
  return LS_OK;
}

ls_status ls_runner_elapsed_ms(ls_runner* r, float* ms) {
  if (!r || !ms) {
    set_error("ls_runner_elapsed_ms: bad arguments");
    return LS_ERR_ARG;
  }
  *ms = r->last_ms;
  return LS_OK;
}

ls_status ls_runner_launch_count(ls_runner* r, int64_t* count) {
  if (!r || !count) {
    set_error("ls_runner_launch_count: bad arguments");
    return LS_ERR_ARG;
  }
  *count = r->launches;
  return LS_OK;
}

ls_status ls_runner_trace_tc(ls_runner* r, const char* program, size_t len, int launches, uint64_t* out,
                             int max_ctas, int* n_ctas) {
  if (!r || !r->have_workload || !program || !out || !n_ctas || launches < 1) {
    set_error("ls_runner_trace_tc: bad arguments");
    return LS_ERR_ARG;
  }
  std::vector<Plan> plans;
  const char* progs[1] = {program};
  size_t lens[1] = {len};
  plan_all(r->w, r->general ? &r->gw : nullptr, r->lim, progs, lens, 1, &plans,
           r->has_alt ? &r->gw : nullptr);
  Plan& plan = plans[0];
  int ctas = 0;
  if (plan.status == P_OK && plan.family == F_TC && !plan.gp) {
    ctas = static_cast<int>(plan.tc.grid_m * plan.tc.grid_n * plan.tc.batch * plan.tc.splits);
  } else if (plan.status == P_OK && plan.gp) {
    for (const GStep& stp : plan.gp->steps)
      if (stp.family == F_TCCONV) ctas = static_cast<int>(stp.conv.grid_m * stp.conv.grid_n * stp.conv.splits);
  }
  if (!ctas) {
    set_error("ls_runner_trace_tc: program does not instantiate as a tcgen05 candidate");
    return LS_ERR_ARG;
  }
  if (plan.gp) {  // general workloads: bytecode of this one candidate
    LSB_CUDA(cudaSetDevice(r->device));
    const std::vector<int64_t>& code = plan.gp->gen.code;
    if (code.size() > r->gcode_cap) {
      cudaFree(r->gcode);
      r->gcode = nullptr;
      r->gcode_cap = std::max(code.size(), 2 * r->gcode_cap);
      LSB_CUDA(cudaMalloc(&r->gcode, r->gcode_cap * 8));
    }
    if (!code.empty()) LSB_CUDA(cudaMemcpy(r->gcode, code.data(), code.size() * 8, cudaMemcpyHostToDevice));
    plan.gcode = r->gcode;
  }
  *n_ctas = ctas;
  LSB_CUDA(cudaSetDevice(r->device));
  unsigned long long* d = nullptr;
  LSB_CUDA(cudaMalloc(&d, static_cast<size_t>(ctas) * 8 * 8 * launches));
  LSB_CUDA(cudaMemsetAsync(d, 0, static_cast<size_t>(ctas) * 8 * 8 * launches, r->st));
  ls_status ps = r->prepare_sync(plans);
  if (ps != LS_OK) {
    cudaFree(d);
    return ps;
  }
  // the launches are captured into one CUDA graph and replayed back to back,
  // as the runner's timed repeats (PDL-chained, no host gaps)
  bool ok = cudaStreamBeginCapture(r->cap_st, cudaStreamCaptureModeThreadLocal) == cudaSuccess;
  for (int i = 0; i < launches && ok; ++i) {
    r->trace = d + static_cast<size_t>(i) * ctas * 8;
    ok = r->launch(plan, false, 0, r->cap_st);
  }
  r->trace = nullptr;
  cudaGraph_t g = nullptr;
  cudaGraphExec_t ge = nullptr;
  const cudaError_t ce = cudaStreamEndCapture(r->cap_st, &g);
  ok = ok && ce == cudaSuccess && g && cudaGraphInstantiate(&ge, g, 0) == cudaSuccess;
  if (g) cudaGraphDestroy(g);
  cudaEvent_t t0 = nullptr, t1 = nullptr;
  cudaEventCreate(&t0);
  cudaEventCreate(&t1);
  if (ok) ok = cudaGraphUpload(ge, r->st) == cudaSuccess && cudaEventRecord(t0, r->st) == cudaSuccess &&
               cudaGraphLaunch(ge, r->st) == cudaSuccess && cudaEventRecord(t1, r->st) == cudaSuccess;
  cudaError_t e = cudaStreamSynchronize(r->st);
  if (ok && e == cudaSuccess) cudaEventElapsedTime(&r->last_ms, t0, t1);  // ls_runner_elapsed_ms: the traced graph
  cudaEventDestroy(t0);
  cudaEventDestroy(t1);
  if (ge) cudaGraphExecDestroy(ge);
  if (!ok) cudaGetLastError();
  int keep = std::min(max_ctas, ctas * launches);
  if (ok && e == cudaSuccess)
    e = cudaMemcpy(out, d, static_cast<size_t>(keep) * 8 * 8, cudaMemcpyDeviceToHost);
  cudaFree(d);
  if (!ok || e != cudaSuccess) {
    set_error("ls_runner_trace_tc: launch failed");
    return LS_ERR_CUDA;
  }
  return LS_OK;
}

ls_status ls_runner_debug_stats(ls_runner* r, double* out, int n) {
  if (!r || !out) {
    set_error("ls_runner_debug_stats: bad arguments");
    return LS_ERR_ARG;
  }
  const double override_us = n > 7 ? out[7] : 0.0;  // optional override (us per call)
  for (int i = 0; i < n && i < 8; ++i) out[i] = r->stats[i];
  if (override_us > 0) r->launch_host_us = override_us;
  return LS_OK;
}

ls_status ls_runner_set_timeout(ls_runner* r, double timeout_ms) {
  if (!r || !(timeout_ms > 0.0)) {
    set_error("ls_runner_set_timeout: bad arguments");
    return LS_ERR_ARG;
  }
  r->opts.timeout_ms = timeout_ms;
  return LS_OK;
}

void ls_runner_destroy(ls_runner* r) { delete r; }

}  // extern "C"
