// Device-side cost-model types and launchers (K7, K8).  See costmodel.cu.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace lsb {

// MachineSpec (`src/machine.py:22-55`); unroll_discount as an exact fraction.
struct DSpec {
  long long cores, vector_lanes, cache_capacity, hit_cost, miss_cost, flop_cost, tensor_unit_cost;
  long long unroll_num, unroll_den;
};

// CostModel parameters (`src/costmodel.py:82-102`).
struct DModel {
  double w[9], mean[9], scale[9], intercept;
  long long n_records;
  int is_fit;
};

// `predict_features`: exp(((f - mean) / scale) . w + intercept); unfit models
// predict exp(intercept) when warm-started, else 1.
__host__ __device__ inline double score_one(const double* f, const DModel& m) {
  if (!m.is_fit) return m.n_records ? exp(m.intercept) : 1.0;
  double dot = 0.0;
  for (int i = 0; i < 9; ++i) dot += ((f[i] - m.mean[i]) / m.scale[i]) * m.w[i];
  return exp(dot + m.intercept);
}

void launch_analyze(const int64_t* blobs, const int64_t* offsets, int n, const DSpec& spec, const DModel& model,
                    int flags, int64_t* lat_num, int64_t* lat_den, double* feats, double* pred, int* status,
                    cudaStream_t stream);
void launch_score(const double* feats, int n, const DModel& model, double* out, cudaStream_t stream);

}  // namespace lsb
