// Flat per-program descriptors for the batched cost kernels (K7 featurize +
// score, K8 exact simulated latency).  The encoder does only syntactic work
// (name resolution, access lists, bytecode for index expressions, which
// enclosing loop drives which access); every cost computation -- interval
// footprints, cache-suffix search, miss classification, exact rational
// latency, the 9 features and the linear score -- runs on the GPU.
//
// One program = one contiguous blob of int64 words (layout below).  A batch
// is the concatenation of blobs plus an offsets array.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "ir.hpp"

namespace lsb {

// blob header
constexpr int H_NLOOP = 0, H_NSTMT = 1, H_NBUF = 2, H_OFF_LOOP = 3, H_OFF_BUF = 4, H_OFF_STMT = 5,
              H_WORDS = 6, H_STATUS = 7, HDR_WORDS = 8;
// loop record
constexpr int L_EXTENT = 0, L_KIND = 1, L_DEPTH = 2, L_PARENT = 3, LOOP_WORDS = 4;
// buffer record: ndim, shape[7]
constexpr int MAX_DIM = 7, BUF_WORDS = 1 + MAX_DIM;
// statement record
constexpr int S_TYPE = 0, S_NL = 1, S_OFF_ENC = 2, S_FLOPS = 3, S_INIT_OPS = 4, S_EPI_OPS = 5,
              S_HAS_INIT = 6, S_HAS_EPI = 7, S_RED_MASK = 8, S_VF_OK = 9, S_NACC = 10, S_OFF_ACC = 11,
              S_TILE0 = 12, S_IFLOPS = 13, S_IOPEL = 14, STMT_WORDS = 16;
// access record: buf, phase, ndim, tile, use_mask, code offsets per dim
constexpr int A_BUF = 0, A_PHASE = 1, A_NDIM = 2, A_TILE = 3, A_USE = 4, A_CODE = 5,
              ACC_WORDS = A_CODE + MAX_DIM;
// bytecode: [n_ops] then n_ops pairs (op, arg); VAR arg = enclosing position
constexpr int BC_INT = 0, BC_VAR = 1, BC_ADD = 2, BC_SUB = 3, BC_MUL = 4, BC_MAX = 5, BC_MIN = 6,
              BC_FDIV = 7, BC_MOD = 8, BC_SEL = 9;
constexpr int MAX_NEST = 62;     // masks are 64-bit
constexpr int MAX_BUFS = 16;
constexpr int MAX_STACK = 24;

// Encodes one program (already parsed).  Returns false with `err` on limits.
bool encode_cost_blob(const Program& p, std::vector<int64_t>* out, std::string* err);

}  // namespace lsb
