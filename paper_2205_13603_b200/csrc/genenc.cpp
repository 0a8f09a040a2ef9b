// Encoder for the generic block executor (see generic.hpp).
#include "generic.hpp"

#include <algorithm>

namespace lsb {

namespace {

struct GenEnc {
  const Program& p;
  GenProgram* out;
  std::string* err;

  bool fail(const char* m) {
    if (err && err->empty()) *err = m;
    return false;
  }

  bool emit(const Expr* e, const std::vector<Stmt*>& loops, std::vector<int64_t>* ops) {
    switch (e->op) {
      case Op::Int:
        ops->push_back(G_CONST);
        ops->push_back(e->value);
        return true;
      case Op::Var:
        for (size_t i = 0; i < loops.size(); ++i)
          if (loops[i]->var == e->var) {
            ops->push_back(G_VAR);
            ops->push_back(static_cast<int64_t>(i));
            return true;
          }
        return fail("expression uses a variable that is not an enclosing loop");
      case Op::Load:
        for (const Expr* k : e->kids)
          if (!emit(k, loops, ops)) return false;
        ops->push_back(G_LOAD);
        ops->push_back(static_cast<int64_t>(e->buffer) | (static_cast<int64_t>(e->kids.size()) << 32));
        return true;
      default:
        break;
    }
    for (const Expr* k : e->kids)
      if (!emit(k, loops, ops)) return false;
    int64_t op = 0;
    switch (e->op) {
      case Op::Add: op = G_ADD; break;
      case Op::Sub: op = G_SUB; break;
      case Op::Mul: op = G_MUL; break;
      case Op::Max: op = G_MAX; break;
      case Op::Min: op = G_MIN; break;
      case Op::FloorDiv: op = G_FDIV; break;
      case Op::Mod: op = G_MOD; break;
      case Op::Select: op = G_SEL; break;
      default: return fail("unsupported expression op");
    }
    ops->push_back(op);
    ops->push_back(0);
    return true;
  }

  int64_t expr(const Expr* e, const std::vector<Stmt*>& loops) {
    std::vector<int64_t> ops;
    if (!emit(e, loops, &ops)) return -1;
    int64_t at = static_cast<int64_t>(out->code.size());
    out->code.push_back(static_cast<int64_t>(ops.size() / 2));
    out->code.insert(out->code.end(), ops.begin(), ops.end());
    return at;
  }
};

}  // namespace

bool encode_generic(const Program& p, GenProgram* out, std::string* err) {
  if (p.buffers.size() > static_cast<size_t>(kGenMaxBufs)) {
    if (err) *err = "too many buffers";
    return false;
  }
  out->blocks.clear();
  out->code.clear();
  out->nbuf = static_cast<int>(p.buffers.size());
  for (size_t b = 0; b < p.buffers.size(); ++b) {
    if (p.buffers[b].shape.size() > 8) {
      if (err) *err = "buffer rank above 8";
      return false;
    }
    out->ndim[b] = static_cast<int>(p.buffers[b].shape.size());
    for (size_t d = 0; d < p.buffers[b].shape.size(); ++d) out->shape[b][d] = p.buffers[b].shape[d];
  }
  GenEnc enc{p, out, err};
  for (const Block& blk : blocks_preorder(p)) {
    const Stmt* s = blk.stmt;
    if (s->type != SType::Compute) {
      if (err) *err = "intrinsic blocks are not executable by the generic executor";
      return false;
    }
    if (blk.loops.size() > static_cast<size_t>(kGenMaxLoops) || s->indices.size() > 8) {
      if (err) *err = "block nest too deep";
      return false;
    }
    GenBlock g;
    g.nl = static_cast<int>(blk.loops.size());
    std::vector<int> store_vars, used;
    for (const Expr* e : s->indices) expr_vars(e, &store_vars);
    expr_vars(s->value, &used);
    if (s->init) expr_vars(s->init, &used);
    for (int i = 0; i < g.nl; ++i) {
      const Stmt* l = blk.loops[static_cast<size_t>(i)];
      g.ext[i] = l->extent;
      bool red = s->init && std::find(used.begin(), used.end(), l->var) != used.end() &&
                 std::find(store_vars.begin(), store_vars.end(), l->var) == store_vars.end();
      if (red) {
        g.red_mask |= 1u << i;
        g.red_trip *= l->extent;
      } else {
        g.points *= l->extent;
      }
    }
    g.store_buf = s->buffer;
    g.store_ndim = static_cast<int>(s->indices.size());
    for (size_t d = 0; d < s->indices.size(); ++d)
      if ((g.store_code[d] = enc.expr(s->indices[d], blk.loops)) < 0) return false;
    if ((g.value_code = enc.expr(s->value, blk.loops)) < 0) return false;
    if (s->init && (g.init_code = enc.expr(s->init, blk.loops)) < 0) return false;
    if (s->epilogue && (g.epi_code = enc.expr(s->epilogue, blk.loops)) < 0) return false;
    out->blocks.push_back(g);
  }
  return true;
}

}  // namespace lsb
