// Encoder for the cost-kernel descriptors.  See costdesc.hpp for the layout.
// Access order follows the reference's `_accesses` (`src/machine.py:66-84`);
// the vector-friendliness rule is `_vector_friendly` (`src/machine.py:177-202`).
#include "costdesc.hpp"

#include <algorithm>

namespace lsb {

namespace {

struct Enc {
  const Program& p;
  std::vector<int64_t>& w;
  std::string* err;
  std::vector<int64_t> loops;   // LOOP_WORDS each
  std::vector<int64_t> stmts;   // STMT_WORDS each
  std::vector<int64_t> tail;    // enc arrays, accesses, bytecode (offsets patched later)
  // tail-relative offsets to patch: positions in stmts/accs that hold tail offsets
  std::vector<size_t> stmt_tail_fix;  // index into stmts
  std::vector<size_t> tail_tail_fix;  // index into tail
  std::vector<int> loop_of_var;       // var id -> loop index
  std::vector<Stmt*> loop_nodes;

  bool fail(const std::string& m) { if (err && err->empty()) *err = m; return false; }

  bool code(const Expr* e, const std::vector<Stmt*>& enc, std::vector<int64_t>* ops) {
    switch (e->op) {
      case Op::Int: ops->push_back(BC_INT); ops->push_back(e->value); return true;
      case Op::Var: {
        for (size_t pos = 0; pos < enc.size(); ++pos)
          if (enc[pos]->var == e->var) { ops->push_back(BC_VAR); ops->push_back(static_cast<int64_t>(pos)); return true; }
        return fail("index uses a variable that is not an enclosing loop");
      }
      case Op::Load: return fail("data-dependent index expression");
      default: break;
    }
    for (const Expr* k : e->kids)
      if (!code(k, enc, ops)) return false;
    int bc = 0;
    switch (e->op) {
      case Op::Add: bc = BC_ADD; break;
      case Op::Sub: bc = BC_SUB; break;
      case Op::Mul: bc = BC_MUL; break;
      case Op::Max: bc = BC_MAX; break;
      case Op::Min: bc = BC_MIN; break;
      case Op::FloorDiv: bc = BC_FDIV; break;
      case Op::Mod: bc = BC_MOD; break;
      case Op::Select: bc = BC_SEL; break;
      default: return fail("bad op");
    }
    ops->push_back(bc);
    ops->push_back(0);
    return true;
  }

  // An index bytecode built from constants, loop variables, +, - and
  // products with a constant side, as c0 + sum coef * var with one term per
  // variable OCCURRENCE (never merged).  Interval arithmetic over such a tree
  // (`src/ir.py:394-433`) equals the sum of the per-term intervals
  // [min(0, coef * E), max(0, coef * E)] plus c0 exactly -- scaling by a
  // constant distributes over interval sums -- so K7 evaluates it as a short
  // loop instead of interpreting the stack code.  Output: c0, then
  // (position, coef) pairs.
  static bool affine_form(const std::vector<int64_t>& ops, std::vector<int64_t>* out) {
    struct Lin {
      int64_t c0 = 0;
      std::vector<std::pair<int64_t, int64_t>> t;
    };
    std::vector<Lin> st;
    for (size_t i = 0; i + 1 < ops.size(); i += 2) {
      const int64_t op = ops[i], arg = ops[i + 1];
      if (op == BC_INT) { st.push_back(Lin{arg, {}}); continue; }
      if (op == BC_VAR) { st.push_back(Lin{0, {{arg, 1}}}); continue; }
      if (st.size() < 2) return false;
      Lin b = std::move(st.back());
      st.pop_back();
      Lin a = std::move(st.back());
      st.pop_back();
      if (op == BC_SUB) {
        b.c0 = -b.c0;
        for (auto& q : b.t) q.second = -q.second;
      }
      if (op == BC_ADD || op == BC_SUB) {
        a.c0 += b.c0;
        a.t.insert(a.t.end(), b.t.begin(), b.t.end());
        st.push_back(std::move(a));
      } else if (op == BC_MUL) {
        if (!a.t.empty() && !b.t.empty()) return false;
        Lin& v = a.t.empty() ? b : a;
        const int64_t k = a.t.empty() ? a.c0 : b.c0;
        v.c0 *= k;
        for (auto& q : v.t) q.second *= k;
        st.push_back(std::move(v));
      } else {
        return false;
      }
    }
    if (st.size() != 1 || st[0].t.size() > 32) return false;
    out->clear();
    out->push_back(st[0].c0);
    for (const auto& q : st[0].t) {
      out->push_back(q.first);
      out->push_back(q.second);
    }
    return true;
  }

  uint64_t use_mask(const std::vector<Expr*>& idx, const std::vector<Stmt*>& enc) {
    std::vector<int> vs;
    for (const Expr* e : idx) expr_vars(e, &vs);
    uint64_t m = 0;
    for (int v : vs)
      for (size_t pos = 0; pos < enc.size(); ++pos)
        if (enc[pos]->var == v) m |= 1ull << pos;
    return m;
  }

  // vector-friendliness of this statement for each enclosing position
  uint64_t vf_ok(const Stmt* s, const std::vector<Stmt*>& enc) {
    std::vector<const std::vector<Expr*>*> lists;
    std::vector<const Expr*> lds;
    if (s->type == SType::Compute) {
      collect_loads(s->value, &lds);
      for (const Expr* l : lds) lists.push_back(&l->kids);
      lists.push_back(&s->indices);
      lds.clear();
      if (s->init) collect_loads(s->init, &lds);
      if (s->epilogue) collect_loads(s->epilogue, &lds);
      for (const Expr* l : lds) lists.push_back(&l->kids);
    } else {
      for (const auto& ix : s->op_indices) lists.push_back(&ix);
    }
    // per index list, once: its variables, the variables of every dimension
    // but the last, and the last dimension's affine coefficients; then each
    // enclosing position is a few lookups
    struct ListInfo {
      std::vector<int> all, lead;
      bool affine = false;
      std::vector<int64_t> coeff;
    };
    std::vector<ListInfo> info(lists.size());
    for (size_t k = 0; k < lists.size(); ++k) {
      const auto* ix = lists[k];
      ListInfo& li = info[k];
      for (const Expr* e : *ix) expr_vars(e, &li.all);
      for (size_t d = 0; d + 1 < ix->size(); ++d) expr_vars((*ix)[d], &li.lead);
      int64_t c0;
      li.affine = !ix->empty() && affine_coeffs(ix->back(), p.vars.size(), &li.coeff, &c0);
    }
    uint64_t ok = 0;
    for (size_t pos = 0; pos < enc.size(); ++pos) {
      int v = enc[pos]->var;
      bool good = true;
      for (const ListInfo& li : info) {
        if (std::find(li.all.begin(), li.all.end(), v) == li.all.end()) continue;
        if (std::find(li.lead.begin(), li.lead.end(), v) != li.lead.end()) good = false;
        if (!li.affine || li.coeff[v] != 1) good = false;
        if (!good) break;
      }
      if (good) ok |= 1ull << pos;
    }
    return ok;
  }

  bool stmt(Stmt* s, std::vector<Stmt*>* enc) {
    if (s->type == SType::Loop) {
      if (enc->size() >= static_cast<size_t>(MAX_NEST)) return fail("loop nest deeper than limit");
      int idx = static_cast<int>(loops.size() / LOOP_WORDS);
      loops.push_back(s->extent);
      loops.push_back(static_cast<int64_t>(s->kind));
      loops.push_back(static_cast<int64_t>(enc->size()));
      int parent = -1;
      if (!enc->empty()) {
        for (size_t li = 0; li < loop_nodes.size(); ++li)
          if (loop_nodes[li] == enc->back()) parent = static_cast<int>(li);
      }
      loops.push_back(parent);
      loop_nodes.push_back(s);
      (void)idx;
      enc->push_back(s);
      for (Stmt* c : s->body)
        if (!stmt(c, enc)) return false;
      enc->pop_back();
      return true;
    }
    size_t rec = stmts.size();
    stmts.resize(rec + STMT_WORDS, 0);
    auto at = [&](int k) -> int64_t& { return stmts[rec + k]; };
    at(S_TYPE) = s->type == SType::Compute ? 0 : 1;
    at(S_NL) = static_cast<int64_t>(enc->size());
    // enclosing loop indices
    at(S_OFF_ENC) = static_cast<int64_t>(tail.size());
    stmt_tail_fix.push_back(rec + S_OFF_ENC);
    for (Stmt* l : *enc)
      for (size_t li = 0; li < loop_nodes.size(); ++li)
        if (loop_nodes[li] == l) tail.push_back(static_cast<int64_t>(li));
    at(S_VF_OK) = static_cast<int64_t>(vf_ok(s, *enc));
    if (s->type == SType::Intrinsic) {
      int n = 0;
      const IntrinsicInfo& info = intrinsic_registry(&n)[s->intrinsic];
      at(S_TILE0) = info.tile0;
      at(S_IFLOPS) = info.flops;
      at(S_IOPEL) = info.operand_elements;
      return emit_accesses(s, *enc, rec);
    }
    std::vector<int> store_vars, used;
    for (const Expr* e : s->indices) expr_vars(e, &store_vars);
    expr_vars(s->value, &used);
    if (s->init) expr_vars(s->init, &used);
    uint64_t red = 0;
    if (s->init)
      for (size_t pos = 0; pos < enc->size(); ++pos) {
        int v = (*enc)[pos]->var;
        bool u = std::find(used.begin(), used.end(), v) != used.end();
        bool st = std::find(store_vars.begin(), store_vars.end(), v) != store_vars.end();
        if (u && !st) red |= 1ull << pos;
      }
    at(S_RED_MASK) = static_cast<int64_t>(red);
    at(S_FLOPS) = arith_ops(s->value) + (s->init ? 1 : 0);
    at(S_INIT_OPS) = s->init ? arith_ops(s->init) : 0;
    at(S_EPI_OPS) = s->epilogue ? arith_ops(s->epilogue) : 0;
    at(S_HAS_INIT) = s->init != nullptr;
    at(S_HAS_EPI) = s->epilogue != nullptr;
    return emit_accesses(s, *enc, rec);
  }

  // Access records are written contiguously (ACC_WORDS apart) followed by
  // their bytecode; we therefore build them in a scratch encoder.
  bool emit_accesses(Stmt* s, const std::vector<Stmt*>& enc, size_t rec) {
    struct A { int buf; const std::vector<Expr*>* idx; int phase; int tile; };
    std::vector<A> list;
    if (s->type == SType::Intrinsic) {
      int n = 0;
      const IntrinsicInfo& info = intrinsic_registry(&n)[s->intrinsic];
      for (size_t i = 0; i < s->op_buffers.size(); ++i)
        list.push_back({s->op_buffers[i], &s->op_indices[i], 0, info.tile0});
    } else {
      std::vector<const Expr*> lds;
      collect_loads(s->value, &lds);
      for (const Expr* l : lds) list.push_back({l->buffer, &l->kids, 0, 1});
      list.push_back({s->buffer, &s->indices, 0, 1});
      if (s->init) {
        list.push_back({s->buffer, &s->indices, 0, 1});
        lds.clear();
        collect_loads(s->init, &lds);
        for (const Expr* l : lds) list.push_back({l->buffer, &l->kids, 1, 1});
        list.push_back({s->buffer, &s->indices, 1, 1});
      }
      if (s->epilogue) {
        lds.clear();
        collect_loads(s->epilogue, &lds);
        for (const Expr* l : lds) list.push_back({l->buffer, &l->kids, 2, 1});
        list.push_back({s->buffer, &s->indices, 2, 1});
      }
    }
    if (list.size() > 64) return fail("too many accesses in one statement");
    stmts[rec + S_NACC] = static_cast<int64_t>(list.size());
    stmts[rec + S_OFF_ACC] = static_cast<int64_t>(tail.size());
    stmt_tail_fix.push_back(rec + S_OFF_ACC);
    size_t first = tail.size();
    tail.resize(first + list.size() * ACC_WORDS, 0);
    for (size_t a = 0; a < list.size(); ++a) {
      size_t r = first + a * ACC_WORDS;
      const A& x = list[a];
      if (x.idx->size() > static_cast<size_t>(MAX_DIM)) return fail("buffer rank above limit");
      if (x.buf < 0 || x.buf >= MAX_BUFS) return fail("buffer count above limit");
      tail[r + A_BUF] = x.buf;
      tail[r + A_PHASE] = x.phase;
      tail[r + A_NDIM] = static_cast<int64_t>(x.idx->size());
      tail[r + A_TILE] = x.tile;
      tail[r + A_USE] = static_cast<int64_t>(use_mask(*x.idx, enc));
      for (size_t d = 0; d < x.idx->size(); ++d) {
        std::vector<int64_t> ops;
        if (!code((*x.idx)[d], enc, &ops)) return false;
        if (ops.size() / 2 > 64) return fail("index expression too long");
        size_t c = tail.size();
        std::vector<int64_t> lin;
        if (affine_form(ops, &lin)) {  // [-(terms + 1), c0, (pos, coef) x terms]
          tail.push_back(-static_cast<int64_t>((lin.size() - 1) / 2) - 1);
          tail.insert(tail.end(), lin.begin(), lin.end());
        } else {
          tail.push_back(static_cast<int64_t>(ops.size() / 2));
          tail.insert(tail.end(), ops.begin(), ops.end());
        }
        tail[r + A_CODE + d] = static_cast<int64_t>(c);
        tail_tail_fix.push_back(r + A_CODE + d);
      }
    }
    return true;
  }
};

}  // namespace

bool encode_cost_blob(const Program& p, std::vector<int64_t>* out, std::string* err) {
  if (p.buffers.size() > static_cast<size_t>(MAX_BUFS)) {
    if (err) *err = "buffer count above limit";
    return false;
  }
  std::vector<int64_t>& w = *out;
  w.clear();
  Enc e{p, w, err};
  std::vector<Stmt*> enc;
  for (Stmt* s : p.root)
    if (!e.stmt(s, &enc)) return false;
  std::sort(e.stmt_tail_fix.begin(), e.stmt_tail_fix.end());
  e.stmt_tail_fix.erase(std::unique(e.stmt_tail_fix.begin(), e.stmt_tail_fix.end()), e.stmt_tail_fix.end());

  int64_t nloop = static_cast<int64_t>(e.loops.size() / LOOP_WORDS);
  int64_t nstmt = static_cast<int64_t>(e.stmts.size() / STMT_WORDS);
  int64_t nbuf = static_cast<int64_t>(p.buffers.size());
  int64_t off_loop = HDR_WORDS;
  int64_t off_buf = off_loop + nloop * LOOP_WORDS;
  int64_t off_stmt = off_buf + nbuf * BUF_WORDS;
  int64_t off_tail = off_stmt + nstmt * STMT_WORDS;
  for (size_t i : e.stmt_tail_fix) e.stmts[i] += off_tail;
  for (size_t i : e.tail_tail_fix) e.tail[i] += off_tail;
  w.resize(static_cast<size_t>(off_tail), 0);
  w[H_NLOOP] = nloop;
  w[H_NSTMT] = nstmt;
  w[H_NBUF] = nbuf;
  w[H_OFF_LOOP] = off_loop;
  w[H_OFF_BUF] = off_buf;
  w[H_OFF_STMT] = off_stmt;
  std::copy(e.loops.begin(), e.loops.end(), w.begin() + off_loop);
  for (int64_t b = 0; b < nbuf; ++b) {
    const Buffer& B = p.buffers[static_cast<size_t>(b)];
    if (B.shape.size() > static_cast<size_t>(MAX_DIM)) {
      if (err) *err = "buffer rank above limit";
      return false;
    }
    w[static_cast<size_t>(off_buf + b * BUF_WORDS)] = static_cast<int64_t>(B.shape.size());
    for (size_t d = 0; d < B.shape.size(); ++d) w[static_cast<size_t>(off_buf + b * BUF_WORDS + 1) + d] = B.shape[d];
  }
  std::copy(e.stmts.begin(), e.stmts.end(), w.begin() + off_stmt);
  w.insert(w.end(), e.tail.begin(), e.tail.end());
  w[H_WORDS] = static_cast<int64_t>(w.size());
  w[H_STATUS] = 0;
  return true;
}

}  // namespace lsb
