// Trace-to-kernel instantiator: maps a final program (the replayed trace's
// TensorProgram) to one kernel family + configuration.  It is a pure function
// of the program (SURVEY.md §7 decision 3): search dedups by structural hash,
// so every kernel knob must be visible in the loop nest.
//
// Mapping convention (replaces the absent `bind`, SURVEY.md §7 decision 4):
//   * every loop of the contraction block is a part of one role axis
//     (batch / M / N / K), recovered from the affine index expressions;
//     adjacent parts of one axis are merged (same iteration order);
//   * any non-serial loop kind            -> LOOPNEST: the parallel loop is the
//     thread index, every other loop runs in order inside the thread;
//   * one part per axis (the unscheduled e0) -> NAIVE: one thread per output;
//   * innermost parts [M 128][N 16..256][K 64] with bf16 data -> TCGEN05:
//     one UMMA tile per CTA, K parts hoisted above every spatial loop become
//     split-K, the other outer K parts the k-tile pipeline, spatial parts the
//     grid; with fp32 data the same tile runs as 3xTF32 (hi/lo operand
//     halves, three kind::tf32 UMMAs per k step, fp32-accurate);
//   * otherwise                            -> SIMT: spatial part 0 -> grid,
//     part 1 -> threads, parts >= 2 -> per-thread register tile; innermost K
//     part -> shared-memory k-tile (BK), outer K parts -> k-tile loop.
// Configurations outside hardware limits are ILLEGAL (the paper's validator
// for "beyond the physical hardware limit").
#pragma once

#include <algorithm>
#include <cstdlib>
#include <cstdint>
#include <memory>
#include <string>
#include <vector>

#include "ir.hpp"

namespace lsb {

enum Role { R_BATCH = 0, R_M = 1, R_N = 2, R_K = 3, R_COUNT = 4 };

// The contraction C[b,m,n] += X[b,m,k] * Y[b,n,k] (any index order/layout)
// recovered from e0.
struct Workload {
  std::string block;               // contraction block name
  int x_buf = -1, y_buf = -1, c_buf = -1;
  int64_t extent[R_COUNT] = {1, 1, 1, 1};
  bool has_batch = false;
  // element strides per role (0 when the role does not index the buffer)
  int64_t sx[R_COUNT] = {0}, sy[R_COUNT] = {0}, sc[R_COUNT] = {0};
  // witness (buffer, dim) whose index is exactly the role variable in e0
  int wit_buf[R_COUNT] = {-1, -1, -1, -1}, wit_dim[R_COUNT] = {-1, -1, -1, -1};
  std::vector<int> input_bufs;     // declared input order
  int64_t x_elems = 0, y_elems = 0, c_elems = 0;
  bool y_kmajor = false;           // K is Y's contiguous dim
  bool x_kmajor = false;
  double flops() const { return 2.0 * extent[0] * extent[1] * extent[2] * extent[3]; }
};

bool analyze_workload(const Program& e0, Workload* w, std::string* err);

enum Family { F_NONE = 0, F_NAIVE = 1, F_SIMT = 2, F_TC = 3, F_LOOPNEST = 4, F_GENERIC = 5, F_NESTGEN = 6, F_SIMTA = 7, F_TCCONV = 8, F_AFFCOPY = 9 };
enum PlanStatus { P_OK = 0, P_ILLEGAL = 1, P_UNSUPPORTED = 2, P_PARSE = 3 };

struct Part { int role; int64_t extent; int64_t stride; Kind kind; };

struct SimtCfg {
  int64_t gb, gm, gn;     // grid
  int64_t tb, tm, tn;     // threads
  int64_t rb, rm, rn;     // per-thread tile (rb looped)
  int64_t bk, kt;         // smem k-tile, k-tiles
  int64_t smem_bytes;
};

struct TcCfg {
  int64_t bn, splits, kt, grid_m, grid_n, batch;
  int64_t stages, smem_bytes;  // stages: ring slots (3xTF32: 32-element k sub-tiles, two per k-tile)
  bool x3 = false;              // fp32 workload: 3xTF32 operand halves
};

// Split-K reduction of the TCGEN05 family and the shared-memory layout it
// implies (tc_gemm.cu).
//   mode 0: splits == 1   single CTA per tile, plain stores
//   mode 2: L2 reduction  the first CTA of the tile to start zeroes it (its
//                         loads are in flight), every split adds its partial
//                         (TMA add-reduce) once the zeroing is released; the
//                         arrival ticket per tile also gives each launch its
//                         own epoch, so there is no memset node between
//                         launches
//   mode 3: mode 2 beyond kTcSyncSlots tiles: fp32 atomics into a memset C
// Measured and dropped (profiles/r01b_summary.md §1, profiles/r02_gemm_lab.md):
// cluster reduce-scatter through DSMEM (~20 B/clk per SM, below the L2 add
// rate), TMA multicast of A across N-tiles (L2 already dedups concurrent
// reads), a store-first epilogue without zeroing, early zero-flag polling.
constexpr int kTcSyncSlots = 4096;  // ticket slots per candidate (mode 2)
struct TcGeom {
  int mode = 0;
  bool tma_epi = false;     // BN % 32 == 0: 128B-swizzled 32-column chunks, TMA store / add-reduce
  bool direct = false;      // mode 0, BN <= 32: TMEM -> registers -> global, no staging
  int ld = 0;               // padded fp32 row of the staged tile (generic epilogue)
  int64_t stage_bytes = 0;  // one stage: A 128 rows + B BN rows of 128 bytes (bf16 k-tile of 64;
                            // 3xTF32: hi and lo of a 32-element fp32 k sub-tile, twice the bytes)
  int64_t ring = 0, tile = 0, smem = 0;
};
inline TcGeom tc_geom(int64_t bn, int64_t splits, int64_t stages, int64_t tiles, bool x3 = false) {
  TcGeom g;
  g.mode = splits == 1 ? 0 : tiles <= kTcSyncSlots ? 2 : 3;
  // no split and a narrow tile: each thread stores its TMEM row straight from
  // registers (bmm QK^T BN 16: 2.08 vs 2.40 us staged, profiles/r02_gemm_lab.md §5)
  g.direct = g.mode == 0 && bn <= 32;
  g.tma_epi = bn % 32 == 0 && g.mode != 3 && !g.direct;
  g.ld = static_cast<int>(bn + 4);  // padded fp32 row (16-byte aligned, conflict-free)
  g.stage_bytes = (128 * 64 * 2 + bn * 64 * 2) * (x3 ? 2 : 1);
  g.ring = stages * g.stage_bytes;
  // staged accumulator tile, overlays the finished ring
  g.tile = g.direct ? 0 : g.tma_epi ? (bn / 32) * 16384 : 128LL * g.ld * 4;
  g.smem = 1024 + std::max(g.ring, g.tile) + 256;
  return g;
}

constexpr int kMaxLoopNest = 16;
struct LoopNestCfg {
  int n;
  int64_t ext[kMaxLoopNest];
  int64_t dx[kMaxLoopNest], dy[kMaxLoopNest], dc[kMaxLoopNest];
};

struct Plan {
  int status = P_UNSUPPORTED;
  int family = F_NONE;
  std::string why;
  std::vector<Part> parts;  // merged, nest order
  SimtCfg simt{};
  TcCfg tc{};
  LoopNestCfg nest{};
  bool needs_zero = false;  // output accumulated with += (memset first)
  int32_t cfg[13] = {0};    // reporting
  std::shared_ptr<struct GeneralPlan> gp;  // general workloads: block-by-block steps
  const int64_t* gcode = nullptr;          // device copy of gp->gen.code
};

struct DeviceLimits {
  int64_t max_threads = 1024;
  int64_t max_smem = 227 * 1024;
  bool bf16 = false;    // runner dtype bf16 and the tcgen05 operand layout available
  bool tf32x3 = false;  // runner dtype fp32 and the 3xTF32 operand halves available
};

Plan plan_program(const Workload& w, const Program& p, const DeviceLimits& lim);

// Register-tile lattice compiled ahead of time for the SIMT family: every
// RM x RN <= 64 over {1,2,3,4,6,8,12,16,24,32,48,64} (the 2^a 3^b divisors
// of the BERT / ResNet extents).
constexpr int kSimtTiles = 12;
bool simt_tile_supported(int64_t rm, int64_t rn);
int simt_tile_index(int64_t v);  // index into the lattice or -1

}  // namespace lsb
