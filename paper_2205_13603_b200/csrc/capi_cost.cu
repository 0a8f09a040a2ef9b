// C-ABI: batched cost model (K7) and exact simulator (K8).
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <mutex>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/loopsched_b200.h"
#include "common.hpp"
#include "costdesc.hpp"
#include "costmodel.cuh"
#include "ir.hpp"

namespace lsb {

namespace {
thread_local std::string g_error;
}

void set_error(const std::string& msg) { g_error = msg; }
const char* last_error() { return g_error.c_str(); }

namespace {

DSpec to_dspec(const ls_machine_spec* s) {
  DSpec d;
  d.cores = s->cores;
  d.vector_lanes = s->vector_lanes;
  d.cache_capacity = s->cache_capacity;
  d.hit_cost = s->hit_cost;
  d.miss_cost = s->miss_cost;
  d.flop_cost = s->flop_cost;
  d.tensor_unit_cost = s->tensor_unit_cost;
  d.unroll_num = s->unroll_num;
  d.unroll_den = s->unroll_den;
  return d;
}

DModel to_dmodel(const ls_linear_model* m) {
  DModel d;
  std::memset(&d, 0, sizeof d);
  if (!m) return d;
  for (int i = 0; i < 9; ++i) {
    d.w[i] = m->w[i];
    d.mean[i] = m->mean[i];
    d.scale[i] = m->scale[i];
  }
  d.intercept = m->intercept;
  d.n_records = m->n_records;
  d.is_fit = m->is_fit;
  return d;
}

ls_status use_device(int device) {
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
    cudaGetLastError();
    set_error("no CUDA device: the B200 path has no CPU fallback");
    return LS_ERR_CUDA;
  }
  if (device < 0 || device >= count) {
    set_error("device index out of range");
    return LS_ERR_ARG;
  }
  LSB_CUDA(cudaSetDevice(device));
  return LS_OK;
}

}  // namespace

}  // namespace lsb

using namespace lsb;

struct ls_batch {
  int device = 0;
  int n = 0;
  cudaStream_t stream = nullptr;
  int64_t* d_blobs = nullptr;
  int64_t* d_off = nullptr;
  int64_t* d_num = nullptr;
  int64_t* d_den = nullptr;
  double* d_feats = nullptr;
  double* d_pred = nullptr;
  int32_t* d_status = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  size_t words = 0;
};

extern "C" {

const char* ls_last_error(void) { return lsb::last_error(); }
const char* ls_version(void) { return "loopsched_b200 0.1 (sm_100a)"; }

ls_status ls_batch_create(int device, const char* const* programs, const size_t* lens, int n, ls_batch** out) {
  if (!out || n < 0 || (n > 0 && (!programs || !lens))) {
    set_error("ls_batch_create: bad arguments");
    return LS_ERR_ARG;
  }
  ls_status st = use_device(device);
  if (st != LS_OK) return st;
  // host: parse + encode (threads), then one upload
  std::vector<std::vector<int64_t>> blobs(static_cast<size_t>(n));
  parallel_for(n, [&](int i) {
    std::string err;
    auto p = parse_program(std::string_view(programs[i], lens[i]), &err);
    std::vector<int64_t>& b = blobs[static_cast<size_t>(i)];
    if (!p) {
      b.assign(HDR_WORDS, 0);
      b[H_STATUS] = LS_PROG_PARSE;
      return;
    }
    if (!encode_cost_blob(*p, &b, &err)) {
      b.assign(HDR_WORDS, 0);
      b[H_STATUS] = LS_PROG_ANALYSIS;
    }
  });
  std::vector<int64_t> offsets(static_cast<size_t>(n) + 1, 0);
  for (int i = 0; i < n; ++i) offsets[i + 1] = offsets[i] + static_cast<int64_t>(blobs[i].size());
  std::vector<int64_t> flat(static_cast<size_t>(offsets[n] > 0 ? offsets[n] : 1));
  for (int i = 0; i < n; ++i) std::copy(blobs[i].begin(), blobs[i].end(), flat.begin() + offsets[i]);

  auto* b = new ls_batch();
  b->device = device;
  b->n = n;
  b->words = flat.size();
  auto fail = [&](cudaError_t e) {
    set_error(std::string("ls_batch_create: ") + cudaGetErrorString(e));
    ls_batch_destroy(b);
    return LS_ERR_CUDA;
  };
  cudaError_t e;
  size_t nn = static_cast<size_t>(n > 0 ? n : 1);
  if ((e = cudaStreamCreateWithFlags(&b->stream, cudaStreamNonBlocking)) != cudaSuccess) return fail(e);
  if ((e = cudaMalloc(&b->d_blobs, flat.size() * 8)) != cudaSuccess) return fail(e);
  if ((e = cudaMalloc(&b->d_off, (nn + 1) * 8)) != cudaSuccess) return fail(e);
  if ((e = cudaMalloc(&b->d_num, nn * 8)) != cudaSuccess) return fail(e);
  if ((e = cudaMalloc(&b->d_den, nn * 8)) != cudaSuccess) return fail(e);
  if ((e = cudaMalloc(&b->d_feats, nn * 9 * 8)) != cudaSuccess) return fail(e);
  if ((e = cudaMalloc(&b->d_pred, nn * 8)) != cudaSuccess) return fail(e);
  if ((e = cudaMalloc(&b->d_status, nn * 4)) != cudaSuccess) return fail(e);
  if ((e = cudaEventCreate(&b->ev0)) != cudaSuccess) return fail(e);
  if ((e = cudaEventCreate(&b->ev1)) != cudaSuccess) return fail(e);
  if ((e = cudaMemcpyAsync(b->d_blobs, flat.data(), flat.size() * 8, cudaMemcpyHostToDevice, b->stream)) != cudaSuccess)
    return fail(e);
  if ((e = cudaMemcpyAsync(b->d_off, offsets.data(), (static_cast<size_t>(n) + 1) * 8, cudaMemcpyHostToDevice,
                           b->stream)) != cudaSuccess)
    return fail(e);
  if ((e = cudaStreamSynchronize(b->stream)) != cudaSuccess) return fail(e);
  *out = b;
  return LS_OK;
}

ls_status ls_batch_analyze(ls_batch* b, const ls_machine_spec* spec, const ls_linear_model* model, int flags) {
  if (!b || !spec) {
    set_error("ls_batch_analyze: bad arguments");
    return LS_ERR_ARG;
  }
  LSB_CUDA(cudaSetDevice(b->device));
  if (!model) flags &= ~4;
  LSB_CUDA(cudaEventRecord(b->ev0, b->stream));
  launch_analyze(b->d_blobs, b->d_off, b->n, to_dspec(spec), to_dmodel(model), flags, b->d_num, b->d_den,
                 b->d_feats, b->d_pred, b->d_status, b->stream);
  LSB_CUDA(cudaGetLastError());
  LSB_CUDA(cudaEventRecord(b->ev1, b->stream));
  return LS_OK;
}

ls_status ls_batch_results(ls_batch* b, int64_t* num, int64_t* den, double* feats, double* pred, int32_t* status) {
  if (!b) {
    set_error("ls_batch_results: null batch");
    return LS_ERR_ARG;
  }
  LSB_CUDA(cudaSetDevice(b->device));
  size_t n = static_cast<size_t>(b->n);
  if (num) LSB_CUDA(cudaMemcpyAsync(num, b->d_num, n * 8, cudaMemcpyDeviceToHost, b->stream));
  if (den) LSB_CUDA(cudaMemcpyAsync(den, b->d_den, n * 8, cudaMemcpyDeviceToHost, b->stream));
  if (feats) LSB_CUDA(cudaMemcpyAsync(feats, b->d_feats, n * 9 * 8, cudaMemcpyDeviceToHost, b->stream));
  if (pred) LSB_CUDA(cudaMemcpyAsync(pred, b->d_pred, n * 8, cudaMemcpyDeviceToHost, b->stream));
  if (status) LSB_CUDA(cudaMemcpyAsync(status, b->d_status, n * 4, cudaMemcpyDeviceToHost, b->stream));
  LSB_CUDA(cudaStreamSynchronize(b->stream));
  return LS_OK;
}

ls_status ls_batch_elapsed_ms(ls_batch* b, float* ms) {
  if (!b || !ms) {
    set_error("ls_batch_elapsed_ms: bad arguments");
    return LS_ERR_ARG;
  }
  LSB_CUDA(cudaEventSynchronize(b->ev1));
  LSB_CUDA(cudaEventElapsedTime(ms, b->ev0, b->ev1));
  return LS_OK;
}

void ls_batch_destroy(ls_batch* b) {
  if (!b) return;
  cudaSetDevice(b->device);
  if (b->stream) cudaStreamSynchronize(b->stream);
  cudaFree(b->d_blobs);
  cudaFree(b->d_off);
  cudaFree(b->d_num);
  cudaFree(b->d_den);
  cudaFree(b->d_feats);
  cudaFree(b->d_pred);
  cudaFree(b->d_status);
  if (b->ev0) cudaEventDestroy(b->ev0);
  if (b->ev1) cudaEventDestroy(b->ev1);
  if (b->stream) cudaStreamDestroy(b->stream);
  delete b;
}

namespace {

// One persistent, growable device workspace per device for the one-shot
// entry points (the search calls them once per new program, so per-call
// allocation would dominate).
struct Workspace {
  std::mutex mu;
  cudaStream_t stream = nullptr;
  // one device block in ([n + 1 offsets][blob words]) and one out
  // ([num n][den n][feats 9n][pred n][status n int32]), laid out per call
  // exactly like the pinned host staging, so a call is one H2D copy, the
  // kernel and one D2H copy (the search calls this once per new program)
  int64_t* d_in = nullptr;
  uint8_t* d_out = nullptr;
  int64_t* h_in = nullptr;
  uint8_t* h_out = nullptr;
  size_t cap_in = 0, cap_out = 0;  // words / bytes
};
Workspace g_ws[64];

inline size_t out_bytes(size_t n) { return n * (8 + 8 + 72 + 8 + 4); }

ls_status grow(Workspace& w, size_t in_words, size_t n) {
  if (!w.stream) LSB_CUDA(cudaStreamCreateWithFlags(&w.stream, cudaStreamNonBlocking));
  if (in_words > w.cap_in) {
    cudaFree(w.d_in);
    cudaFreeHost(w.h_in);
    w.d_in = nullptr;
    w.h_in = nullptr;
    const size_t c = std::max(in_words, 2 * w.cap_in);
    LSB_CUDA(cudaMalloc(&w.d_in, c * 8));
    LSB_CUDA(cudaMallocHost(&w.h_in, c * 8));
    w.cap_in = c;
  }
  if (out_bytes(n) > w.cap_out) {
    cudaFree(w.d_out);
    cudaFreeHost(w.h_out);
    w.d_out = nullptr;
    w.h_out = nullptr;
    const size_t c = std::max(out_bytes(n), 2 * w.cap_out);
    LSB_CUDA(cudaMalloc(&w.d_out, c));
    LSB_CUDA(cudaMallocHost(&w.h_out, c));
    w.cap_out = c;
  }
  return LS_OK;
}

}  // namespace

ls_status ls_analyze_batch(int device, const char* const* programs, const size_t* lens, int n,
                           const ls_machine_spec* spec, const ls_linear_model* model, int64_t* num, int64_t* den,
                           double* feats, double* pred, int32_t* status) {
  if (!spec || n < 0 || (n > 0 && (!programs || !lens))) {
    set_error("ls_analyze_batch: bad arguments");
    return LS_ERR_ARG;
  }
  ls_status st = use_device(device);
  if (st != LS_OK) return st;
  if (device >= 64) {
    set_error("ls_analyze_batch: device index above 63");
    return LS_ERR_ARG;
  }
  if (n == 0) return LS_OK;
  std::vector<std::vector<int64_t>> blobs(static_cast<size_t>(n));
  parallel_for(n, [&](int i) {
    std::string err;
    auto p = parse_program(std::string_view(programs[i], lens[i]), &err);
    std::vector<int64_t>& b = blobs[static_cast<size_t>(i)];
    if (!p) {
      b.assign(HDR_WORDS, 0);
      b[H_STATUS] = LS_PROG_PARSE;
    } else if (!encode_cost_blob(*p, &b, &err)) {
      b.assign(HDR_WORDS, 0);
      b[H_STATUS] = LS_PROG_ANALYSIS;
    }
  });
  const size_t nn = static_cast<size_t>(n);
  std::vector<int64_t> offsets(nn + 1, 0);
  for (int i = 0; i < n; ++i) offsets[i + 1] = offsets[i] + static_cast<int64_t>(blobs[i].size());
  const size_t words = static_cast<size_t>(offsets[nn]);

  Workspace& w = g_ws[device];
  std::lock_guard<std::mutex> lock(w.mu);
  if ((st = grow(w, nn + 1 + words, nn)) != LS_OK) return st;
  // offsets then the blobs, contiguous in pinned memory: one DMA
  int64_t* hin = w.h_in;
  std::copy(offsets.begin(), offsets.end(), hin);
  int64_t* hblob = hin + nn + 1;
  parallel_for(n, [&](int i) {
    std::copy(blobs[static_cast<size_t>(i)].begin(), blobs[static_cast<size_t>(i)].end(), hblob + offsets[i]);
  });
  LSB_CUDA(cudaMemcpyAsync(w.d_in, hin, (nn + 1 + words) * 8, cudaMemcpyHostToDevice, w.stream));
  int64_t* d_num = reinterpret_cast<int64_t*>(w.d_out);
  int64_t* d_den = d_num + nn;
  double* d_feats = reinterpret_cast<double*>(d_den + nn);
  double* d_pred = d_feats + 9 * nn;
  int32_t* d_status = reinterpret_cast<int32_t*>(d_pred + nn);
  int flags = (num || den ? 1 : 0) | (feats ? 2 : 0) | (pred && model ? 4 : 0);
  launch_analyze(w.d_in + nn + 1, w.d_in, n, to_dspec(spec), to_dmodel(model), flags, d_num, d_den, d_feats,
                 d_pred, d_status, w.stream);
  LSB_CUDA(cudaGetLastError());
  LSB_CUDA(cudaMemcpyAsync(w.h_out, w.d_out, out_bytes(nn), cudaMemcpyDeviceToHost, w.stream));
  LSB_CUDA(cudaStreamSynchronize(w.stream));
  int64_t* o_num = reinterpret_cast<int64_t*>(w.h_out);
  int64_t* o_den = o_num + nn;
  double* o_feats = reinterpret_cast<double*>(o_den + nn);
  double* o_pred = o_feats + 9 * nn;
  int32_t* o_status = reinterpret_cast<int32_t*>(o_pred + nn);
  if (num) std::memcpy(num, o_num, nn * 8);
  if (den) std::memcpy(den, o_den, nn * 8);
  if (feats) std::memcpy(feats, o_feats, nn * 72);
  if (pred && model) std::memcpy(pred, o_pred, nn * 8);
  if (status) std::memcpy(status, o_status, nn * 4);
  return LS_OK;
}

ls_status ls_sim_latency_batch(int device, const char* const* programs, const size_t* lens, int n,
                               const ls_machine_spec* spec, int64_t* num, int64_t* den, int32_t* status) {
  if (!num || !den) {
    set_error("ls_sim_latency_batch: null output");
    return LS_ERR_ARG;
  }
  return ls_analyze_batch(device, programs, lens, n, spec, nullptr, num, den, nullptr, nullptr, status);
}

ls_status ls_featurize_batch(int device, const char* const* programs, const size_t* lens, int n,
                             const ls_machine_spec* spec, double* feats, int32_t* status) {
  if (!feats) {
    set_error("ls_featurize_batch: null output");
    return LS_ERR_ARG;
  }
  return ls_analyze_batch(device, programs, lens, n, spec, nullptr, nullptr, nullptr, feats, nullptr, status);
}

ls_status ls_score_batch(int device, const double* feats, int n, const ls_linear_model* model, double* out) {
  if (!feats || !model || !out || n < 0) {
    set_error("ls_score_batch: bad arguments");
    return LS_ERR_ARG;
  }
  ls_status st = use_device(device);
  if (st != LS_OK) return st;
  if (n == 0) return LS_OK;
  if (device >= 64) {
    set_error("ls_score_batch: device index above 63");
    return LS_ERR_ARG;
  }
  Workspace& w = g_ws[device];
  std::lock_guard<std::mutex> lock(w.mu);
  const size_t nn = static_cast<size_t>(n);
  if ((st = grow(w, 9 * nn, nn)) != LS_OK) return st;
  double* d_feats = reinterpret_cast<double*>(w.d_in);
  double* d_pred = reinterpret_cast<double*>(w.d_out);
  LSB_CUDA(cudaMemcpyAsync(d_feats, feats, nn * 72, cudaMemcpyHostToDevice, w.stream));
  launch_score(d_feats, n, to_dmodel(model), d_pred, w.stream);
  LSB_CUDA(cudaGetLastError());
  LSB_CUDA(cudaMemcpyAsync(out, d_pred, nn * 8, cudaMemcpyDeviceToHost, w.stream));
  LSB_CUDA(cudaStreamSynchronize(w.stream));
  return LS_OK;
}

}  // extern "C"
