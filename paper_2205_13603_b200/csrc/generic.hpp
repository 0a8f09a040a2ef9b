// Generic block executor: any Compute block of any program, evaluated from
// postfix bytecode on the GPU.  One thread per point of the block's non-
// reduction loops (in nest order); the thread runs the block's reduction loops
// in nest order with init on the first and epilogue on the last iteration --
// the statement semantics of the reference interpreter (`src/interp.py:
// 184-244`, `:388-467`).  Used for the reference output of any workload
// (fp64), for the unscheduled baseline of multi-block workloads, and for
// elementwise blocks (pad stages) of candidate programs.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "ir.hpp"

namespace lsb {

// bytecode ops (pairs of int64: op, arg)
enum GenOp : int64_t {
  G_CONST = 0, G_VAR = 1, G_LOAD = 2, G_ADD = 3, G_SUB = 4, G_MUL = 5, G_MAX = 6, G_MIN = 7,
  G_FDIV = 8, G_MOD = 9, G_SEL = 10
};
// LOAD arg = buffer id | (ndim << 32); pops ndim index values, pushes value.
// An out-of-range load yields 0 without touching memory (only reachable in the
// untaken branch of a Select guard in valid programs).

constexpr int kGenMaxLoops = 24;
constexpr int kGenMaxBufs = 16;

struct GenBlock {
  int nl = 0;
  int64_t ext[kGenMaxLoops] = {0};
  uint32_t red_mask = 0;     // loops that carry the reduction (run inside a thread)
  int store_buf = -1;
  int store_ndim = 0;
  // offsets into the code vector
  int64_t store_code[8] = {0};
  int64_t value_code = -1, init_code = -1, epi_code = -1;
  int64_t points = 1;        // product of non-reduction extents
  int64_t red_trip = 1;
};

struct GenProgram {
  std::vector<GenBlock> blocks;
  std::vector<int64_t> code;  // [n_ops, op, arg, op, arg, ...] per expression
  int nbuf = 0;
  int64_t shape[kGenMaxBufs][8] = {{0}};
  int ndim[kGenMaxBufs] = {0};
};

bool encode_generic(const Program& p, GenProgram* out, std::string* err);

// AFFCOPY: an elementwise stage whose value is a load (optionally behind the
// load's own in-bounds Select guard, i.e. a pad) whose indices are
// quasi-affine in the block's loop variables: sums of c * ((v / d) % m)
// terms, which covers split (affine), fuse (floordiv / mod of the fused
// variable, `src/schedule.py:374-382`) and their compositions.
//   out[sum_out] = all guards in range ? in[sum_in] : 0
constexpr int kCopyMaxLoops = 12;
constexpr int kCopyMaxGuard = 4;
constexpr int kQMax = 16;
struct QTerm { int32_t loop, div, mod, pad; int64_t coef; };
struct QSum {
  int n = 0;
  int64_t c0 = 0;
  QTerm t[kQMax];
};
struct CopyCfg {
  int nl = 0, ng = 0;
  int in_buf = -1, out_buf = -1;
  int64_t ext[kCopyMaxLoops] = {0};
  QSum out, in;                 // element offsets
  QSum g[kCopyMaxGuard];        // guarded input dims (index values)
  int64_t gext[kCopyMaxGuard] = {0};
  int64_t points = 1;
  // innermost loops that walk both buffers contiguously (coef 1, run, ...)
  // and no guard: one thread copies `vec` consecutive elements of that run
  int run_loops = 0;        // how many innermost loops form the run
  int64_t run = 1;          // elements per run
  int vec = 1;              // elements per thread (divides run)
};

}  // namespace lsb
