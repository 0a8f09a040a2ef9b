// Program model for the B200 path: the reference IR (`src/ir.py:25-175`)
// parsed from its fixed-schema JSON interchange format (`src/ir.py:671-815`).
//
// This is the native front end of the C-ABI: everything crossing the
// boundary is the reference's own serialized program text, so a caller can
// hand over `ir.serialize(program)` unchanged.
#pragma once

#include <cstdint>
#include <memory>
#include <string>
#include <string_view>
#include <vector>

namespace lsb {

enum class Op : uint8_t { Int, Var, Load, Add, Sub, Mul, Max, Min, FloorDiv, Mod, Select };

struct Expr {
  Op op = Op::Int;
  int64_t value = 0;           // Int
  int var = -1;                // Var: program-wide var id
  int buffer = -1;             // Load
  std::vector<Expr*> kids;     // binop: a,b ; select: cond,then,other ; load: indices
};

enum class Kind : uint8_t { Serial, Parallel, Vectorized, Unrolled };
enum class SType : uint8_t { Loop, Compute, Intrinsic };

struct Stmt {
  SType type = SType::Loop;
  // loop
  int var = -1;
  int64_t extent = 0;
  Kind kind = Kind::Serial;
  std::vector<Stmt*> body;
  // compute / intrinsic
  std::string name;            // block name
  int buffer = -1;             // compute store buffer
  std::vector<Expr*> indices;  // compute store indices
  Expr* value = nullptr;
  Expr* init = nullptr;
  Expr* epilogue = nullptr;
  int intrinsic = -1;          // index into intrinsic registry
  std::vector<int> op_buffers;             // intrinsic operands
  std::vector<std::vector<Expr*>> op_indices;
};

struct Buffer {
  std::string name;
  std::vector<int64_t> shape;
  int role = 0;  // 0 input, 1 output, 2 intermediate
};

// Intrinsic registry of `src/schedule.py:40-42`.
struct IntrinsicInfo {
  const char* name;
  int tile0;
  int64_t flops;
  int64_t operand_elements;
};
const IntrinsicInfo* intrinsic_registry(int* n);

// Node storage: fixed-size chunks, so a parse costs one allocation per chunk
// instead of one per node (nodes never move; freed with the program).
template <class T, size_t kChunk>
struct NodeArena {
  std::vector<std::unique_ptr<T[]>> chunks;
  size_t used = kChunk;
  T* alloc() {
    if (used == kChunk) {
      chunks.emplace_back(new T[kChunk]);
      used = 0;
    }
    return &chunks.back()[used++];
  }
};

struct Program {
  std::vector<Buffer> buffers;
  std::vector<std::string> vars;  // var id -> name
  std::vector<Stmt*> root;
  // ownership
  NodeArena<Expr, 64> expr_pool;
  NodeArena<Stmt, 16> stmt_pool;

  int buffer_id(std::string_view name) const;
  Expr* new_expr() { return expr_pool.alloc(); }
  Stmt* new_stmt() { return stmt_pool.alloc(); }
};

// Parses `text`; on failure returns nullptr and fills `err`.
std::unique_ptr<Program> parse_program(std::string_view text, std::string* err);

// ---- analysis helpers ------------------------------------------------------

// A statement together with its enclosing loops (outer -> inner), pre-order.
struct Block {
  Stmt* stmt;
  std::vector<Stmt*> loops;
};
std::vector<Block> blocks_preorder(const Program& p);

void expr_vars(const Expr* e, std::vector<int>* out);  // appends (may repeat)
int64_t arith_ops(const Expr* e);                        // `src/ir.py:436-445`
void collect_loads(const Expr* e, std::vector<const Expr*>* out);  // `src/ir.py:448-465`

// Affine decomposition (`src/ir.py:339-372`): coeff per var id (dense, sized
// to p.vars.size()) and constant; false when not affine.
bool affine_coeffs(const Expr* e, size_t nvars, std::vector<int64_t>* coeff, int64_t* c0);

}  // namespace lsb
