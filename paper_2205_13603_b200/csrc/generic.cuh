// Generic block executor launcher.  See generic.hpp.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "generic.hpp"

namespace lsb {

// Device views of every buffer of a program: dtype 0 bf16, 1 f32, 2 f64.
struct GenBuffers {
  void* ptr[kGenMaxBufs];
  int dtype[kGenMaxBufs];
  int64_t shape[kGenMaxBufs][8];
};

// One kernel for one block; fp64 accumulates in double (reference output).
bool launch_generic_block(const GenBlock& g, const int64_t* code, const GenBuffers& B, bool fp64,
                          const unsigned long long* deadline, int* timed_out, cudaStream_t st);

// PVU structure: thread per iteration of the outermost (parallel) loop.
bool launch_generic_nest(const GenBlock& g, const int64_t* code, const GenBuffers& B,
                         const unsigned long long* deadline, int* timed_out, cudaStream_t st);

// AFFCOPY family (affine elementwise copy / pad), thread per point.
bool launch_affcopy(const CopyCfg& c, const GenBuffers& B, const unsigned long long* deadline, int* timed_out,
                    cudaStream_t st);

}  // namespace lsb
