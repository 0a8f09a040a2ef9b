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
// predict exp(intercept) when warm-started, else 1.  Every operation is
// rounded on its own (no FMA contraction) and the dot product is summed in
// index order; numpy's `z @ w` goes through the BLAS ddot kernel of the host,
// whose summation order (and libm's exp) can differ in the last ulp, so this
// is within ~1e-15 relative of the reference, not bit-identical.  Parity
// mode re-derives the scores the search compares with the reference's own
// formula on the host (plugin.ScoreCache(exact=True)).
__host__ __device__ inline double score_one(const double* f, const DModel& m) {
  if (!m.is_fit) return m.n_records ? exp(m.intercept) : 1.0;
  double dot = 0.0;
#ifdef __CUDA_ARCH__
  for (int i = 0; i < 9; ++i) dot = __dadd_rn(dot, __dmul_rn(__ddiv_rn(__dsub_rn(f[i], m.mean[i]), m.scale[i]), m.w[i]));
  return exp(__dadd_rn(dot, m.intercept));
#else
  for (int i = 0; i < 9; ++i) {
    volatile double z = (f[i] - m.mean[i]) / m.scale[i];
    volatile double p = z * m.w[i];
    dot += p;
  }
  return exp(dot + m.intercept);
#endif
}

void launch_analyze(const int64_t* blobs, const int64_t* offsets, int n, const DSpec& spec, const DModel& model,
                    int flags, int64_t* lat_num, int64_t* lat_den, double* feats, double* pred, int* status,
                    cudaStream_t stream);
void launch_score(const double* feats, int n, const DModel& model, double* out, cudaStream_t stream);

}  // namespace lsb
