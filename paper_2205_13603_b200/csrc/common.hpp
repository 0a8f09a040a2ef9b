// Error plumbing shared by the C-ABI translation units.
#pragma once

#include <cuda_runtime.h>

#include <string>

namespace lsb {

void set_error(const std::string& msg);
const char* last_error();

#define LSB_CUDA(expr)                                                                      \
  do {                                                                                      \
    cudaError_t e_ = (expr);                                                                \
    if (e_ != cudaSuccess) {                                                                \
      ::lsb::set_error(std::string(#expr) + ": " + cudaGetErrorString(e_));                 \
      return LS_ERR_CUDA;                                                                   \
    }                                                                                       \
  } while (0)

// Parse + encode work is spread over host threads (the GPU kernels need the
// descriptors of a whole batch at once).
template <class F>
void parallel_for(int n, F&& f);

}  // namespace lsb

#include <thread>
#include <vector>

namespace lsb {
template <class F>
void parallel_for(int n, F&& f) {
  unsigned hw = std::thread::hardware_concurrency();
  int nt = static_cast<int>(hw ? hw : 4);
  if (nt > 16) nt = 16;
  if (n < 64 || nt <= 1) {
    for (int i = 0; i < n; ++i) f(i);
    return;
  }
  if (nt > n) nt = n;
  std::vector<std::thread> th;
  th.reserve(static_cast<size_t>(nt));
  for (int t = 0; t < nt; ++t)
    th.emplace_back([&, t] {
      for (int i = t; i < n; i += nt) f(i);
    });
  for (auto& x : th) x.join();
}
}  // namespace lsb
