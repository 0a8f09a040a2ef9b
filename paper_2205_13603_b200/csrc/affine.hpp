// General workloads (conv2d NHWC with its pad stage, dense_relu, ...): any
// program whose blocks are elementwise stages plus exactly one contraction
// C[...] (+)= X[...] * Y[...] whose indices are affine sums of loop variables
// (implicit GEMM).  A candidate runs block by block in program order:
//   * elementwise blocks          -> GENERIC (thread per point, bytecode)
//   * contraction, any parallel   -> NESTGEN (PVU structure: thread per
//                                    iteration of the outermost parallel loop)
//   * contraction, one part/axis  -> GENERIC (the unscheduled e0)
//   * contraction, MLT structure  -> SIMT-A: affine SIMT tile kernel whose
//                                    operand addresses come from per-part
//                                    address coefficients (tables built per
//                                    CTA); an inlined pad `Select(guard,
//                                    X[...], 0)` becomes a predicated load
//   * contraction epilogue        -> extra GENERIC pass over the output
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "generic.hpp"
#include "ir.hpp"

namespace lsb {

enum AGroup { AG_M = 0, AG_N = 1, AG_K = 2, AG_B = 3 };
enum ALevel { AL_GRID = 0, AL_THREAD = 1, AL_REG = 2, AL_KTILE = 3, AL_BK = 4 };

struct GeneralWorkload {
  std::string block;                       // contraction block name
  std::vector<std::string> axis_var;       // e0 loop var names of the contraction
  std::vector<int> axis_group;             // AGroup per axis
  std::vector<int64_t> axis_extent;
  // witness per axis: (buffer name, dim) indexed by exactly that variable
  std::vector<std::string> wit_buf;
  std::vector<int> wit_dim;
  std::string x_buf, y_buf, c_buf;         // operand buffer names in e0
  std::vector<std::string> buffers;        // e0 buffer names (device allocations)
  std::vector<std::vector<int64_t>> shapes;
  std::vector<int> roles;                  // 0 input, 1 output, 2 intermediate
  int64_t c_elems = 0;
};

bool analyze_general(const Program& e0, GeneralWorkload* w, std::string* err);

constexpr int kAMaxParts = 24;

struct APart {
  int64_t extent;
  int32_t group, level;
  int64_t cx, cy, cc;   // address coefficient (elements) in X-side, Y, C per unit of this loop
  int64_t cg[2];        // coefficient in the guarded X dims
};

struct AffineCfg {
  int nparts;
  APart parts[kAMaxParts];  // nest order
  int64_t x0, y0, c0;       // constant address terms
  int ng;                   // guarded X dims (inlined pad), <= 2
  int64_t g0[2], gext[2];
  int64_t gm, gn, tm, tn, rm, rn, bk, kt;
  int64_t smem_bytes;
};

// TCGEN05 implicit-GEMM conv: one 8x8 output-pixel box (64 rows, the upper
// half of a 128-row UMMA tile) x BN output channels x 64 input channels per
// k-tile.  Per-part contributions to the TMA coordinates of the 4-D X-side
// box (n, h, w, c), to the flattened K index of the K-major weight copy, and
// to the output address.
constexpr int kConvMaxK = 64;  // splits x k-tiles of one tcgen05 conv candidate
struct CList {
  int n;
  int64_t ext[8], xn[8], xh[8], xw[8], xc[8], kf[8], cc[8], co[8];
};
struct TcConvCfg {
  CList m_grid, n_grid, k_split, k_tile;
  int64_t x_n0, x_h0, x_w0, x_c0;  // constant coordinates (inlined pad: -pad)
  int64_t c0;                      // output address constant
  int64_t cc_h1, cc_w1;            // output address per box row / box column
  int64_t bn, splits, kt, stages, smem_bytes, grid_m, grid_n;
  bool x3;  // fp32 operands as 3xTF32 halves; stages are then 32-channel k sub-tiles (two per k-tile)
};

// Buffer ids of the candidate program, resolved by name against the runner's
// device buffers.
struct GStep {
  int family;               // F_GENERIC, F_NESTGEN, F_SIMTA (plan.hpp Family values)
  int block;                // index into the candidate's GenProgram blocks
  bool epilogue_pass = false;
  AffineCfg aff{};
  TcConvCfg conv{};
  CopyCfg copy{};
  int x_buf = -1, y_buf = -1, c_buf = -1;  // candidate buffer ids (SIMT-A, TC-conv)
  bool x3_split = false;    // 3xTF32 conv on an in-candidate activation: split it into halves each launch
};

struct GeneralPlan {
  int status = 0;           // PlanStatus
  std::string why;
  GenProgram gen;           // candidate blocks as bytecode
  std::vector<std::string> buf_names;  // candidate buffer names
  std::vector<GStep> steps;
  int32_t cfg[13] = {0};
  int family = 0;           // family of the contraction step (reporting)
};

// kernels one launch of a general plan enqueues (a step, plus its per-launch split)
inline int64_t general_kernels(const GeneralPlan& g) {
  int64_t n = 0;
  for (const GStep& s : g.steps) n += s.x3_split ? 2 : 1;
  return n;
}

struct DeviceLimits;
GeneralPlan plan_general(const GeneralWorkload& w, const Program& p, const DeviceLimits& lim);

bool simta_tile_supported(int64_t rm, int64_t rn);
int simta_tile_index(int64_t v);

}  // namespace lsb
