// Native trace replay and validation (follow mode) -- SURVEY.md §8f-1.
//
// Restates, for the search's validator, the reference's
//   * trace replay        `src/trace.py:163-238` (replay / _step / _bind)
//   * validate_trace      `src/trace.py:258-265`
//   * schedule primitives `src/schedule.py:123-974` (ScheduleState: get_blocks,
//     get_loops, split, fuse, reorder, parallelize, vectorize, unroll,
//     compute_at, inline, tensorize and the three samplers in decision-
//     following mode)
//   * IR utilities         `src/ir.py:181-666` (tree navigation, substitution,
//     affine analysis, validate_ir, canonicalize, structural_hash, serialize)
// on an immutable, structurally shared tree (shared_ptr nodes), so one
// primitive costs microseconds instead of the reference's milliseconds.
//
// Outputs are byte-identical to the reference's: the accepted program's
// `ir.serialize` text, its `ir.structural_hash`, and the normalized trace's
// `serialize_trace` text; a rejection carries the reference's
// (reason, instruction index).  Any path on which the reference would raise
// something other than ScheduleError / ReplayError (a malformed trace that
// trips a KeyError/TypeError in Python) is reported as LS_REPLAY_DEFER so the
// caller replays that trace with the reference itself and gets the same
// exception -- behaviour stays identical by construction.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <functional>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <map>
#include <memory>
#include <mutex>
#include <unordered_set>
#include <optional>
#include <set>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <utility>
#include <vector>

#include "../../include/loopsched_b200.h"
#include "common.hpp"
#include "pyjson.hpp"

namespace lsb {
namespace rp {

using pj::Value;

// ---------------------------------------------------------------------------
// IR (src/ir.py:25-175)
// ---------------------------------------------------------------------------

enum EK : uint8_t { E_INT, E_VAR, E_LOAD, E_ADD, E_SUB, E_MUL, E_MAX, E_MIN, E_FDIV, E_MOD, E_SEL };
struct Ex;
using EP = std::shared_ptr<const Ex>;
struct Ex {
  EK k = E_INT;
  int64_t v = 0;
  std::string s;  // Var name / Load buffer
  std::vector<EP> a;
  // memoized analyses of this (immutable, structurally shared) node; a copy
  // starts with empty caches
  mutable int8_t qa = -1;  // is_quasi_affine
  mutable std::shared_ptr<const std::vector<std::string>> vars;  // sorted expr_vars
  Ex() = default;
  Ex(const Ex& o) : k(o.k), v(o.v), s(o.s), a(o.a) {}
};

const char* binop_name(EK k) {
  switch (k) {
    case E_ADD: return "add";
    case E_SUB: return "sub";
    case E_MUL: return "mul";
    case E_MAX: return "max";
    case E_MIN: return "min";
    case E_FDIV: return "floordiv";
    case E_MOD: return "mod";
    default: return nullptr;
  }
}
bool is_binop(EK k) { return k >= E_ADD && k <= E_MOD; }

EP mk_int(int64_t v) {
  auto e = std::make_shared<Ex>();
  e->k = E_INT;
  e->v = v;
  return e;
}
EP mk_var(const std::string& n) {
  auto e = std::make_shared<Ex>();
  e->k = E_VAR;
  e->s = n;
  return e;
}
EP mk_bin(EK k, EP a, EP b) {
  auto e = std::make_shared<Ex>();
  e->k = k;
  e->a = {std::move(a), std::move(b)};
  return e;
}
EP mk_load(const std::string& buf, std::vector<EP> idx) {
  auto e = std::make_shared<Ex>();
  e->k = E_LOAD;
  e->s = buf;
  e->a = std::move(idx);
  return e;
}

bool ex_eq(const EP& x, const EP& y) {
  if (x == y) return true;
  if (!x || !y) return false;
  if (x->k != y->k || x->v != y->v || x->s != y->s || x->a.size() != y->a.size()) return false;
  for (size_t i = 0; i < x->a.size(); ++i)
    if (!ex_eq(x->a[i], y->a[i])) return false;
  return true;
}

enum SKd : uint8_t { S_LOOP, S_COMP, S_INTR };
struct St;
using SP = std::shared_ptr<const St>;
struct St {
  SKd k = S_LOOP;
  // Loop
  std::string var;
  int64_t extent = 0;
  std::string kind;
  std::vector<SP> body;
  // Compute (name, buffer, idx, value, init, epi) / Intrinsic (name, block, ops, init)
  std::string name, buffer, block;
  std::vector<EP> idx;
  EP value, init, epi;
  std::vector<std::pair<std::string, std::vector<EP>>> ops;
};

struct Buf {
  std::string name;
  std::vector<int64_t> shape;
  std::string role;
};
struct Prog {
  std::vector<Buf> bufs;
  std::vector<SP> root;
  const Buf* buffer(const std::string& n) const {
    for (const Buf& b : bufs)
      if (b.name == n) return &b;
    return nullptr;
  }
};
using Path = std::vector<int>;

const std::string& block_name(const St& s) { return s.k == S_COMP ? s.name : s.block; }
bool is_block(const St& s) { return s.k != S_LOOP; }

SP with_body(const St& loop, std::vector<SP> body) {
  auto n = std::make_shared<St>(loop);
  n->body = std::move(body);
  return n;
}
SP mk_loop(const std::string& var, int64_t extent, const std::string& kind, std::vector<SP> body) {
  auto n = std::make_shared<St>();
  n->k = S_LOOP;
  n->var = var;
  n->extent = extent;
  n->kind = kind;
  n->body = std::move(body);
  return n;
}

// ---- exceptions mirroring the reference's control flow ----
struct SchedErr {  // ScheduleError
  std::string msg;
};
struct Defer {  // anything else the reference would raise (caller replays in Python)
  std::string msg;
};
[[noreturn]] void sched_err(std::string m) { throw SchedErr{std::move(m)}; }
[[noreturn]] void defer(std::string m) { throw Defer{std::move(m)}; }

// ---- tree navigation (src/ir.py:181-246) ----
// pre-order (src/ir.py:181-190), children left to right; `f` returns true
// to stop the walk early
template <class F>
bool walk_stmts(const std::vector<SP>& list, Path& path, F& f) {
  for (size_t i = 0; i < list.size(); ++i) {
    path.push_back(static_cast<int>(i));
    if (f(static_cast<const Path&>(path), *list[i])) return true;
    if (list[i]->k == S_LOOP && walk_stmts(list[i]->body, path, f)) return true;
    path.pop_back();
  }
  return false;
}
template <class F>
void iter_stmts(const std::vector<SP>& root, F&& f) {
  Path path;
  auto g = [&](const Path& p, const St& s) {
    f(p, s);
    return false;
  };
  walk_stmts(root, path, g);
}
template <class F>
std::optional<Path> find_first(const std::vector<SP>& root, F&& pred) {
  Path path;
  auto g = [&](const Path&, const St& s) { return pred(s); };
  if (walk_stmts(root, path, g)) return path;
  return std::nullopt;
}

const SP& get_stmt(const std::vector<SP>& root, const Path& path) {
  const SP* s = &root.at(path[0]);
  for (size_t d = 1; d < path.size(); ++d) s = &(*s)->body.at(path[d]);
  return *s;
}

std::vector<SP> replace_stmt(const std::vector<SP>& root, const Path& path, size_t at,
                             const std::vector<SP>& repl) {
  std::vector<SP> out;
  out.reserve(root.size() + repl.size());
  const int i = path[at];
  for (int k = 0; k < i; ++k) out.push_back(root[k]);
  if (at + 1 == path.size()) {
    for (const SP& r : repl) out.push_back(r);
  } else {
    out.push_back(with_body(*root[i], replace_stmt(root[i]->body, path, at + 1, repl)));
  }
  for (size_t k = i + 1; k < root.size(); ++k) out.push_back(root[k]);
  return out;
}
std::vector<SP> replace_stmt(const std::vector<SP>& root, const Path& path, const std::vector<SP>& repl) {
  return replace_stmt(root, path, 0, repl);
}

std::vector<std::pair<Path, SP>> enclosing_loops(const std::vector<SP>& root, const Path& path) {
  std::vector<std::pair<Path, SP>> out;
  const std::vector<SP>* list = &root;
  for (size_t d = 0; d + 1 < path.size(); ++d) {
    const SP& node = (*list)[path[d]];
    out.push_back({Path(path.begin(), path.begin() + d + 1), node});
    list = &node->body;
  }
  return out;
}

std::optional<Path> find_block(const std::vector<SP>& root, const std::string& name) {
  return find_first(root, [&](const St& s) { return is_block(s) && block_name(s) == name; });
}
std::optional<Path> find_loop(const std::vector<SP>& root, const std::string& var) {
  return find_first(root, [&](const St& s) { return s.k == S_LOOP && s.var == var; });
}

// ---- expressions (src/ir.py:253-445) ----
const std::vector<std::string>& var_list(const EP& e) {
  if (!e->vars) {
    auto v = std::make_shared<std::vector<std::string>>();
    if (e->k == E_VAR) {
      v->push_back(e->s);
    } else {
      for (const EP& c : e->a) {
        const auto& cv = var_list(c);
        v->insert(v->end(), cv.begin(), cv.end());
      }
      std::sort(v->begin(), v->end());
      v->erase(std::unique(v->begin(), v->end()), v->end());
    }
    e->vars = std::move(v);
  }
  return *e->vars;
}
void expr_vars(const EP& e, std::set<std::string>* out) {
  if (!e) return;
  const auto& v = var_list(e);
  out->insert(v.begin(), v.end());
}
std::set<std::string> vars_of(const EP& e) {
  std::set<std::string> s;
  expr_vars(e, &s);
  return s;
}
std::set<std::string> vars_of(const std::vector<EP>& es) {
  std::set<std::string> s;
  for (const EP& e : es) expr_vars(e, &s);
  return s;
}

using Subst = std::map<std::string, EP>;
EP substitute(const EP& e, const Subst& m) {
  if (!e) return e;
  if (e->k == E_INT) return e;
  if (e->k == E_VAR) {
    auto it = m.find(e->s);
    return it == m.end() ? e : it->second;
  }
  bool changed = false;
  std::vector<EP> kids;
  kids.reserve(e->a.size());
  for (const EP& c : e->a) {
    kids.push_back(substitute(c, m));
    changed |= kids.back() != c;
  }
  if (!changed) return e;
  auto n = std::make_shared<Ex>(*e);
  n->a = std::move(kids);
  return n;
}
std::vector<EP> substitute(const std::vector<EP>& es, const Subst& m) {
  std::vector<EP> out;
  out.reserve(es.size());
  for (const EP& e : es) out.push_back(substitute(e, m));
  return out;
}
SP substitute_stmt(const SP& s, const Subst& m) {
  auto n = std::make_shared<St>(*s);
  if (s->k == S_LOOP) {
    for (SP& c : n->body) c = substitute_stmt(c, m);
  } else if (s->k == S_COMP) {
    n->idx = substitute(s->idx, m);
    n->value = substitute(s->value, m);
    n->init = substitute(s->init, m);
    n->epi = substitute(s->epi, m);
  } else {
    for (auto& op : n->ops) op.second = substitute(op.second, m);
    n->init = substitute(s->init, m);
  }
  return n;
}

EP rename_loads(const EP& e, const std::string& from, const std::string& to) {
  if (!e || e->k == E_INT || e->k == E_VAR) return e;
  auto n = std::make_shared<Ex>(*e);
  if (e->k == E_LOAD && e->s == from) n->s = to;
  for (EP& c : n->a) c = rename_loads(c, from, to);
  return n;
}

using Coeffs = std::map<std::string, int64_t>;
std::optional<std::pair<Coeffs, int64_t>> affine_coeffs(const EP& e) {
  if (e->k == E_INT) return std::make_pair(Coeffs{}, e->v);
  if (e->k == E_VAR) return std::make_pair(Coeffs{{e->s, 1}}, int64_t{0});
  if (e->k == E_ADD || e->k == E_SUB) {
    auto l = affine_coeffs(e->a[0]);
    auto r = affine_coeffs(e->a[1]);
    if (!l || !r) return std::nullopt;
    const int64_t sign = e->k == E_ADD ? 1 : -1;
    Coeffs c = l->first;
    for (const auto& kv : r->first) {
      c[kv.first] += sign * kv.second;
      if (c[kv.first] == 0) c.erase(kv.first);
    }
    return std::make_pair(std::move(c), l->second + sign * r->second);
  }
  if (e->k == E_MUL) {
    auto l = affine_coeffs(e->a[0]);
    auto r = affine_coeffs(e->a[1]);
    if (!l || !r) return std::nullopt;
    if (!l->first.empty() && !r->first.empty()) return std::nullopt;
    if (!r->first.empty()) std::swap(l, r);
    const int64_t scale = r->second;
    Coeffs c;
    for (const auto& kv : l->first)
      if (kv.second * scale != 0) c[kv.first] = kv.second * scale;
    return std::make_pair(std::move(c), l->second * scale);
  }
  return std::nullopt;
}

bool is_quasi_affine_(const EP& e);
bool is_quasi_affine(const EP& e) {
  if (e->qa < 0) e->qa = is_quasi_affine_(e) ? 1 : 0;
  return e->qa == 1;
}
bool is_quasi_affine_(const EP& e) {
  if (affine_coeffs(e)) return true;
  if (e->k == E_FDIV || e->k == E_MOD)
    return e->a[1]->k == E_INT && e->a[1]->v > 0 && is_quasi_affine(e->a[0]);
  if (e->k == E_MUL) {
    if (e->a[1]->k == E_INT) return is_quasi_affine(e->a[0]);
    if (e->a[0]->k == E_INT) return is_quasi_affine(e->a[1]);
    return false;
  }
  if (e->k == E_ADD || e->k == E_SUB) return is_quasi_affine(e->a[0]) && is_quasi_affine(e->a[1]);
  return false;
}

void collect_loads(const EP& e, std::vector<const Ex*>* out) {
  if (!e) return;
  if (e->k == E_LOAD) {
    out->push_back(e.get());
    for (const EP& i : e->a) collect_loads(i, out);
  } else if (is_binop(e->k) || e->k == E_SEL) {
    for (const EP& c : e->a) collect_loads(c, out);
  }
}

std::string expr_str(const EP& e) {
  switch (e->k) {
    case E_INT: return std::to_string(e->v);
    case E_VAR: return e->s;
    case E_LOAD: {
      std::string s = e->s + "[";
      for (size_t i = 0; i < e->a.size(); ++i) s += (i ? ", " : "") + expr_str(e->a[i]);
      return s + "]";
    }
    case E_SEL:
      return "select(" + expr_str(e->a[0]) + ", " + expr_str(e->a[1]) + ", " + expr_str(e->a[2]) + ")";
    default: {
      const char* sym = e->k == E_ADD ? "+" : e->k == E_SUB ? "-" : e->k == E_MUL ? "*"
                      : e->k == E_FDIV ? "//" : e->k == E_MOD ? "%" : nullptr;
      if (sym) return "(" + expr_str(e->a[0]) + " " + sym + " " + expr_str(e->a[1]) + ")";
      return std::string(binop_name(e->k)) + "(" + expr_str(e->a[0]) + ", " + expr_str(e->a[1]) + ")";
    }
  }
}

std::string py_list_repr(const std::vector<std::string>& xs) {
  std::string s = "[";
  for (size_t i = 0; i < xs.size(); ++i) s += (i ? ", " : "") + pj::py_repr(xs[i]);
  return s + "]";
}
std::string py_int_list(const std::vector<int64_t>& xs) {
  std::string s = "[";
  for (size_t i = 0; i < xs.size(); ++i) s += (i ? ", " : "") + std::to_string(xs[i]);
  return s + "]";
}

// ---- validate_ir (src/ir.py:472-597) ----
std::vector<std::string> stmt_exprs(const St& s) {
  (void)s;
  return {};
}

std::vector<std::string> validate_ir(const Prog& p) {
  std::vector<std::string> diags;
  {
    std::set<std::string> names;
    for (const Buf& b : p.bufs) names.insert(b.name);
    if (names.size() != p.bufs.size()) diags.push_back("duplicate buffer name");
  }
  std::map<std::string, const Buf*> buffers;
  for (const Buf& b : p.bufs) {
    bool bad = b.shape.empty();
    for (int64_t x : b.shape) bad |= x < 1;
    if (bad) diags.push_back("buffer " + b.name + ": shape must be non-empty with positive extents");
    if (b.role != "input" && b.role != "output" && b.role != "intermediate")
      diags.push_back("buffer " + b.name + ": unknown role " + pj::py_repr(b.role));
    buffers[b.name] = &b;
  }
  std::vector<std::string> block_names, loop_vars_seen;
  std::vector<std::pair<std::string, std::vector<std::string>>> writers, readers;  // insertion order
  auto add_to = [](std::vector<std::pair<std::string, std::vector<std::string>>>& m, const std::string& k,
                   const std::string& v) {
    for (auto& kv : m)
      if (kv.first == k) {
        kv.second.push_back(v);
        return;
      }
    m.push_back({k, {v}});
  };
  Path path;
  std::vector<const std::string*> bound_stack;
  std::function<void(const St&)> visit;
  std::function<void(const std::vector<SP>&)> walk = [&](const std::vector<SP>& list) {
    for (size_t i = 0; i < list.size(); ++i) {
      path.push_back(static_cast<int>(i));
      visit(*list[i]);
      if (list[i]->k == S_LOOP) {
        bound_stack.push_back(&list[i]->var);
        walk(list[i]->body);
        bound_stack.pop_back();
      }
      path.pop_back();
    }
  };
  visit = [&](const St& s) {
    // "/".join(path), built only for a diagnostic
    struct Where {
      const Path& p;
      operator std::string() const {
        std::string w;
        for (size_t i = 0; i < p.size(); ++i) w += (i ? "/" : "") + std::to_string(p[i]);
        return w;
      }
    } where_{path};
    auto where = [&]() { return static_cast<std::string>(where_); };
    if (s.k == S_LOOP) {
      if (s.extent < 1) diags.push_back("loop " + s.var + " at " + where() + ": non-positive extent");
      if (s.kind != "serial" && s.kind != "parallel" && s.kind != "vectorized" && s.kind != "unrolled")
        diags.push_back("loop " + s.var + " at " + where() + ": unknown kind " + pj::py_repr(s.kind));
      if (std::find(loop_vars_seen.begin(), loop_vars_seen.end(), s.var) != loop_vars_seen.end())
        diags.push_back("loop " + s.var + " at " + where() + ": duplicate loop variable");
      loop_vars_seen.push_back(s.var);
      return;
    }
    const std::string& name = block_name(s);
    if (std::find(block_names.begin(), block_names.end(), name) != block_names.end())
      diags.push_back("block " + name + " at " + where() + ": duplicate block name");
    block_names.push_back(name);
    struct Bound {
      const std::vector<const std::string*>& st;
      size_t count(const std::string& v) const {
        for (const std::string* x : st)
          if (*x == v) return 1;
        return 0;
      }
    } bound{bound_stack};
    std::vector<EP> exprs;
    if (s.k == S_COMP) {
      exprs = s.idx;
      exprs.push_back(s.value);
      if (s.init) exprs.push_back(s.init);
      if (s.epi) exprs.push_back(s.epi);
    } else {
      for (const auto& op : s.ops) exprs.insert(exprs.end(), op.second.begin(), op.second.end());
      if (s.init) exprs.push_back(s.init);
    }
    for (const EP& e : exprs) {
      const std::vector<std::string>& vs = var_list(e);
      if (vs.size() > 1) {
        // the reference iterates a Python set here: with two or more unbound
        // names the message order is hash-seed dependent
        int unbound = 0;
        for (const auto& v : vs) unbound += !bound.count(v);
        if (unbound > 1) defer("several unbound variables");
      }
      for (const auto& v : vs)
        if (!bound.count(v)) diags.push_back("block " + name + " at " + where() + ": unbound variable " + pj::py_repr(v));
    }
    auto check_access = [&](const std::string& buf, const std::vector<EP>& indices, const char* what) {
      auto it = buffers.find(buf);
      if (it == buffers.end()) {
        diags.push_back("block " + name + " at " + where() + ": " + what + " of undeclared buffer " + pj::py_repr(buf));
        return;
      }
      if (indices.size() != it->second->shape.size())
        diags.push_back("block " + name + " at " + where() + ": " + what + " of " + buf + " has rank " +
                        std::to_string(indices.size()) + ", buffer has rank " +
                        std::to_string(it->second->shape.size()));
      for (const EP& i : indices)
        if (!is_quasi_affine(i))
          diags.push_back("block " + name + " at " + where() + ": non-affine index in " + what + " of " + buf);
    };
    if (s.k == S_COMP) {
      check_access(s.buffer, s.idx, "store");
      add_to(writers, s.buffer, name);
      std::vector<EP> vals{s.value};
      if (s.init) vals.push_back(s.init);
      if (s.epi) vals.push_back(s.epi);
      for (const EP& e : vals) {
        std::vector<const Ex*> lds;
        collect_loads(e, &lds);
        for (const Ex* ld : lds) {
          check_access(ld->s, ld->a, "load");
          if (ld->s != s.buffer) add_to(readers, ld->s, name);
        }
      }
      if (!s.init) {
        std::set<std::string> store = vars_of(s.idx);
        std::vector<std::string> stray;
        for (const auto& v : var_list(s.value))
          if (bound.count(v) && !store.count(v)) stray.push_back(v);  // std::set: sorted
        if (!stray.empty())
          diags.push_back("block " + name + " at " + where() + ": assignment uses loop vars " + py_list_repr(stray) +
                          " absent from its store index (undeclared reduction)");
        if (s.epi) diags.push_back("block " + name + " at " + where() + ": epilogue on a non-reduction block");
      }
    } else {
      if (s.ops.empty()) diags.push_back("intrinsic " + name + " at " + where() + ": no operands");
      for (const auto& op : s.ops) check_access(op.first, op.second, "operand");
      if (!s.ops.empty()) {
        add_to(writers, s.ops[0].first, name);
        for (size_t k = 1; k < s.ops.size(); ++k) add_to(readers, s.ops[k].first, name);
      }
    }
  };
  walk(p.root);
  for (const auto& kv : writers) {
    std::set<std::string> ws(kv.second.begin(), kv.second.end());
    if (ws.size() > 1)
      diags.push_back("buffer " + kv.first + ": written by multiple blocks " +
                      py_list_repr(std::vector<std::string>(ws.begin(), ws.end())));
    auto it = buffers.find(kv.first);
    if (it != buffers.end() && it->second->role == "input")
      diags.push_back("buffer " + kv.first + ": input buffer is written");
  }
  for (const Buf& b : p.bufs) {
    bool written = false;
    for (const auto& kv : writers) written |= kv.first == b.name;
    if (b.role == "output" && !written) diags.push_back("buffer " + b.name + ": output buffer is never written");
  }
  // producer -> consumer acyclicity
  std::map<std::string, std::string> produced_by;
  for (const auto& kv : writers) produced_by[kv.first] = kv.second[0];
  std::map<std::string, std::set<std::string>> edges;
  for (const auto& n : block_names) edges[n];
  for (const auto& kv : readers) {
    auto it = produced_by.find(kv.first);
    if (it == produced_by.end()) continue;
    for (const auto& r : kv.second)
      if (r != it->second) edges[it->second].insert(r);
  }
  std::map<std::string, int> state;
  std::function<bool(const std::string&)> has_cycle = [&](const std::string& n) {
    state[n] = 1;
    for (const auto& m : edges[n]) {
      if (state[m] == 1) return true;
      if (state[m] == 0 && has_cycle(m)) return true;
    }
    state[n] = 2;
    return false;
  };
  for (const auto& n : block_names)
    if (state[n] == 0 && has_cycle(n)) {
      diags.push_back("cyclic producer/consumer dependence involving block " + n);
      break;
    }
  return diags;
}

// ---- serialization (src/ir.py:670-715) and hashing (src/ir.py:605-666) ----
// loop-variable renaming applied by structural_hash while serializing
thread_local const std::unordered_map<std::string, std::string>* g_rename = nullptr;
const std::string& renamed(const std::string& v) {
  if (g_rename) {
    auto it = g_rename->find(v);
    if (it != g_rename->end()) return it->second;
  }
  return v;
}
void ser_expr(const EP& e, std::string* o) {
  switch (e->k) {
    case E_INT: *o += "{\"int\": " + std::to_string(e->v) + "}"; return;
    case E_VAR: *o += "{\"var\": "; pj::dump_string(renamed(e->s), o); *o += "}"; return;
    case E_LOAD:
      *o += "{\"load\": {\"buffer\": ";
      pj::dump_string(e->s, o);
      *o += ", \"indices\": [";
      for (size_t i = 0; i < e->a.size(); ++i) {
        if (i) *o += ", ";
        ser_expr(e->a[i], o);
      }
      *o += "]}}";
      return;
    case E_SEL:
      *o += "{\"select\": [";
      for (int i = 0; i < 3; ++i) {
        if (i) *o += ", ";
        ser_expr(e->a[i], o);
      }
      *o += "]}";
      return;
    default:
      *o += "{\"";
      *o += binop_name(e->k);
      *o += "\": [";
      ser_expr(e->a[0], o);
      *o += ", ";
      ser_expr(e->a[1], o);
      *o += "]}";
      return;
  }
}
void ser_list(const std::vector<EP>& es, std::string* o) {
  *o += "[";
  for (size_t i = 0; i < es.size(); ++i) {
    if (i) *o += ", ";
    ser_expr(es[i], o);
  }
  *o += "]";
}
void ser_stmt(const SP& s, std::string* o) {
  if (s->k == S_LOOP) {
    *o += "{\"loop\": {\"body\": [";
    for (size_t i = 0; i < s->body.size(); ++i) {
      if (i) *o += ", ";
      ser_stmt(s->body[i], o);
    }
    *o += "], \"extent\": " + std::to_string(s->extent) + ", \"kind\": ";
    pj::dump_string(s->kind, o);
    *o += ", \"var\": ";
    pj::dump_string(renamed(s->var), o);
    *o += "}}";
  } else if (s->k == S_COMP) {
    *o += "{\"compute\": {\"buffer\": ";
    pj::dump_string(s->buffer, o);
    if (s->epi) {
      *o += ", \"epilogue\": ";
      ser_expr(s->epi, o);
    }
    *o += ", \"indices\": ";
    ser_list(s->idx, o);
    if (s->init) {
      *o += ", \"init\": ";
      ser_expr(s->init, o);
    }
    *o += ", \"name\": ";
    pj::dump_string(s->name, o);
    *o += ", \"value\": ";
    ser_expr(s->value, o);
    *o += "}}";
  } else {
    *o += "{\"intrinsic\": {\"block\": ";
    pj::dump_string(s->block, o);
    if (s->init) {
      *o += ", \"init\": ";
      ser_expr(s->init, o);
    }
    *o += ", \"name\": ";
    pj::dump_string(s->name, o);
    *o += ", \"operands\": [";
    for (size_t i = 0; i < s->ops.size(); ++i) {
      if (i) *o += ", ";
      *o += "{\"buffer\": ";
      pj::dump_string(s->ops[i].first, o);
      *o += ", \"indices\": ";
      ser_list(s->ops[i].second, o);
      *o += "}";
    }
    *o += "]}}";
  }
}
std::string serialize(const Prog& p) {
  std::string o = "{\"buffers\": [";
  for (size_t i = 0; i < p.bufs.size(); ++i) {
    const Buf& b = p.bufs[i];
    if (i) o += ", ";
    o += "{\"name\": ";
    pj::dump_string(b.name, &o);
    o += ", \"role\": ";
    pj::dump_string(b.role, &o);
    o += ", \"shape\": " + py_int_list(b.shape) + "}";
  }
  o += "], \"root\": [";
  for (size_t i = 0; i < p.root.size(); ++i) {
    if (i) o += ", ";
    ser_stmt(p.root[i], &o);
  }
  o += "]}";
  return o;
}

Prog canonicalize(const Prog& p) {
  std::map<std::string, std::string> mapping;
  iter_stmts(p.root, [&](const Path&, const St& s) {
    if (s.k == S_LOOP && !mapping.count(s.var)) mapping[s.var] = "v" + std::to_string(mapping.size());
  });
  Subst sub;
  for (const auto& kv : mapping) sub[kv.first] = mk_var(kv.second);
  std::function<SP(const SP&)> walk = [&](const SP& s) -> SP {
    if (s->k == S_LOOP) {
      std::vector<SP> body;
      for (const SP& c : s->body) body.push_back(walk(c));
      return mk_loop(mapping[s->var], s->extent, s->kind, std::move(body));
    }
    return substitute_stmt(s, sub);
  };
  Prog q;
  q.bufs = p.bufs;
  for (const SP& s : p.root) q.root.push_back(walk(s));
  return q;
}

// BLAKE2b (RFC 7693), unkeyed, digest_size 8 as in structural_hash
namespace b2 {
const uint64_t IV[8] = {0x6a09e667f3bcc908ULL, 0xbb67ae8584caa73bULL, 0x3c6ef372fe94f82bULL,
                        0xa54ff53a5f1d36f1ULL, 0x510e527fade682d1ULL, 0x9b05688c2b3e6c1fULL,
                        0x1f83d9abfb41bd6bULL, 0x5be0cd19137e2179ULL};
const uint8_t SIGMA[12][16] = {
    {0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15}, {14, 10, 4, 8, 9, 15, 13, 6, 1, 12, 0, 2, 11, 7, 5, 3},
    {11, 8, 12, 0, 5, 2, 15, 13, 10, 14, 3, 6, 7, 1, 9, 4}, {7, 9, 3, 1, 13, 12, 11, 14, 2, 6, 5, 10, 4, 0, 15, 8},
    {9, 0, 5, 7, 2, 4, 10, 15, 14, 1, 11, 12, 6, 8, 3, 13}, {2, 12, 6, 10, 0, 11, 8, 3, 4, 13, 7, 5, 15, 14, 1, 9},
    {12, 5, 1, 15, 14, 13, 4, 10, 0, 7, 6, 3, 9, 2, 8, 11}, {13, 11, 7, 14, 12, 1, 3, 9, 5, 0, 15, 4, 8, 6, 2, 10},
    {6, 15, 14, 9, 11, 3, 0, 8, 12, 2, 13, 7, 1, 4, 10, 5}, {10, 2, 8, 4, 7, 6, 1, 5, 15, 11, 9, 14, 3, 12, 13, 0},
    {0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15}, {14, 10, 4, 8, 9, 15, 13, 6, 1, 12, 0, 2, 11, 7, 5, 3}};
inline uint64_t rotr(uint64_t x, int n) { return (x >> n) | (x << (64 - n)); }
void compress(uint64_t h[8], const uint8_t block[128], uint64_t t, bool last) {
  uint64_t m[16], v[16];
  for (int i = 0; i < 16; ++i) {
    uint64_t x = 0;
    for (int b = 7; b >= 0; --b) x = (x << 8) | block[8 * i + b];
    m[i] = x;
  }
  for (int i = 0; i < 8; ++i) {
    v[i] = h[i];
    v[i + 8] = IV[i];
  }
  v[12] ^= t;
  if (last) v[14] = ~v[14];
  auto G = [&](int a, int b, int c, int d, uint64_t x, uint64_t y) {
    v[a] = v[a] + v[b] + x;
    v[d] = rotr(v[d] ^ v[a], 32);
    v[c] = v[c] + v[d];
    v[b] = rotr(v[b] ^ v[c], 24);
    v[a] = v[a] + v[b] + y;
    v[d] = rotr(v[d] ^ v[a], 16);
    v[c] = v[c] + v[d];
    v[b] = rotr(v[b] ^ v[c], 63);
  };
  for (int r = 0; r < 12; ++r) {
    const uint8_t* s = SIGMA[r];
    G(0, 4, 8, 12, m[s[0]], m[s[1]]);
    G(1, 5, 9, 13, m[s[2]], m[s[3]]);
    G(2, 6, 10, 14, m[s[4]], m[s[5]]);
    G(3, 7, 11, 15, m[s[6]], m[s[7]]);
    G(0, 5, 10, 15, m[s[8]], m[s[9]]);
    G(1, 6, 11, 12, m[s[10]], m[s[11]]);
    G(2, 7, 8, 13, m[s[12]], m[s[13]]);
    G(3, 4, 9, 14, m[s[14]], m[s[15]]);
  }
  for (int i = 0; i < 8; ++i) h[i] ^= v[i] ^ v[i + 8];
}
uint64_t hash8(const std::string& text) {
  uint64_t h[8];
  for (int i = 0; i < 8; ++i) h[i] = IV[i];
  h[0] ^= 0x01010000ULL ^ 8ULL;  // digest length 8, no key
  const uint8_t* p = reinterpret_cast<const uint8_t*>(text.data());
  size_t n = text.size(), off = 0;
  uint8_t block[128];
  while (n - off > 128) {
    compress(h, p + off, static_cast<uint64_t>(off + 128), false);
    off += 128;
  }
  std::memset(block, 0, sizeof block);
  std::memcpy(block, p + off, n - off);
  compress(h, block, static_cast<uint64_t>(n), true);
  uint64_t out = 0;  // first 8 digest bytes (little-endian h[0]) read big-endian
  for (int b = 0; b < 8; ++b) out = (out << 8) | ((h[0] >> (8 * b)) & 0xFF);
  return out;
}
}  // namespace b2

uint64_t structural_hash(const Prog& p) {
  // == blake2b(serialize(canonicalize(p)), 8): the renaming is applied while
  // writing (loop vars in order of first binding; other names unchanged)
  std::unordered_map<std::string, std::string> ren;
  iter_stmts(p.root, [&](const Path&, const St& s) {
    if (s.k == S_LOOP && !ren.count(s.var)) ren.emplace(s.var, "v" + std::to_string(ren.size()));
  });
  g_rename = &ren;
  std::string text;
  try {
    text = serialize(p);
  } catch (...) {
    g_rename = nullptr;
    throw;
  }
  g_rename = nullptr;
  return b2::hash8(text);
}

// ---- deserialize (src/ir.py:718-815): from a parsed JSON document ----
struct BadDoc {};
int64_t as_int(const Value* v) {
  if (!v || v->t != Value::Int || v->big) throw BadDoc{};
  return v->i;
}
const std::string& as_str(const Value* v) {
  if (!v || v->t != Value::Str) throw BadDoc{};
  return v->s;
}
EP expr_from(const Value& d) {
  if (d.t != Value::Obj || d.o.size() != 1) throw BadDoc{};
  const std::string& tag = d.o[0].first;
  const Value& pl = d.o[0].second;
  if (tag == "int") return mk_int(as_int(&pl));
  if (tag == "var") return mk_var(as_str(&pl));
  if (tag == "load") {
    if (pl.t != Value::Obj) throw BadDoc{};
    const Value* idx = pl.get("indices");
    if (!idx || idx->t != Value::Arr) throw BadDoc{};
    std::vector<EP> ix;
    for (const Value& i : idx->a) ix.push_back(expr_from(i));
    return mk_load(as_str(pl.get("buffer")), std::move(ix));
  }
  if (tag == "select") {
    if (pl.t != Value::Arr || pl.a.size() != 3) throw BadDoc{};
    auto e = std::make_shared<Ex>();
    e->k = E_SEL;
    for (const Value& x : pl.a) e->a.push_back(expr_from(x));
    return e;
  }
  static const std::pair<const char*, EK> ops[] = {{"add", E_ADD}, {"sub", E_SUB}, {"mul", E_MUL},
                                                   {"max", E_MAX}, {"min", E_MIN}, {"floordiv", E_FDIV},
                                                   {"mod", E_MOD}};
  for (const auto& op : ops)
    if (tag == op.first) {
      if (pl.t != Value::Arr || pl.a.size() != 2) throw BadDoc{};
      return mk_bin(op.second, expr_from(pl.a[0]), expr_from(pl.a[1]));
    }
  throw BadDoc{};
}
std::vector<EP> exprs_from(const Value* v) {
  if (!v || v->t != Value::Arr) throw BadDoc{};
  std::vector<EP> out;
  for (const Value& x : v->a) out.push_back(expr_from(x));
  return out;
}
SP stmt_from(const Value& d) {
  if (d.t != Value::Obj || d.o.size() != 1) throw BadDoc{};
  const std::string& tag = d.o[0].first;
  const Value& pl = d.o[0].second;
  if (pl.t != Value::Obj) throw BadDoc{};
  auto s = std::make_shared<St>();
  if (tag == "loop") {
    s->k = S_LOOP;
    s->var = as_str(pl.get("var"));
    s->extent = as_int(pl.get("extent"));
    s->kind = as_str(pl.get("kind"));
    const Value* body = pl.get("body");
    if (!body || body->t != Value::Arr) throw BadDoc{};
    for (const Value& c : body->a) s->body.push_back(stmt_from(c));
  } else if (tag == "compute") {
    s->k = S_COMP;
    s->name = as_str(pl.get("name"));
    s->buffer = as_str(pl.get("buffer"));
    s->idx = exprs_from(pl.get("indices"));
    const Value* v = pl.get("value");
    if (!v) throw BadDoc{};
    s->value = expr_from(*v);
    if (const Value* i = pl.get("init"); i && i->t != Value::Null) s->init = expr_from(*i);
    if (const Value* e = pl.get("epilogue"); e && e->t != Value::Null) s->epi = expr_from(*e);
  } else if (tag == "intrinsic") {
    s->k = S_INTR;
    s->name = as_str(pl.get("name"));
    s->block = as_str(pl.get("block"));
    const Value* ops = pl.get("operands");
    if (!ops || ops->t != Value::Arr) throw BadDoc{};
    for (const Value& op : ops->a) {
      if (op.t != Value::Obj) throw BadDoc{};
      s->ops.push_back({as_str(op.get("buffer")), exprs_from(op.get("indices"))});
    }
    if (const Value* i = pl.get("init"); i && i->t != Value::Null) s->init = expr_from(*i);
  } else {
    throw BadDoc{};
  }
  return s;
}
bool program_from(std::string_view text, Prog* p) {
  Value doc;
  if (!pj::parse(text, &doc) || doc.t != Value::Obj) return false;
  try {
    const Value* bufs = doc.get("buffers");
    const Value* root = doc.get("root");
    if (!bufs || !root || bufs->t != Value::Arr || root->t != Value::Arr) return false;
    for (const Value& b : bufs->a) {
      if (b.t != Value::Obj) return false;
      Buf x;
      x.name = as_str(b.get("name"));
      x.role = as_str(b.get("role"));
      const Value* sh = b.get("shape");
      if (!sh || sh->t != Value::Arr) return false;
      for (const Value& e : sh->a) x.shape.push_back(as_int(&e));
      p->bufs.push_back(std::move(x));
    }
    for (const Value& s : root->a) p->root.push_back(stmt_from(s));
  } catch (const BadDoc&) {
    return false;
  }
  return true;
}

// ---------------------------------------------------------------------------
// Schedule state (src/schedule.py:123-974), decision-following mode
// ---------------------------------------------------------------------------

// tu.mma4 of src/schedule.py:40-42
struct IntrInfo {
  const char* name;
  int64_t tile[3];
};
const IntrInfo kIntrinsics[] = {{"tu.mma4", {4, 4, 4}}};
const IntrInfo* intrinsic(const std::string& n) {
  for (const IntrInfo& i : kIntrinsics)
    if (n == i.name) return &i;
  return nullptr;
}

void factorizations(int64_t extent, int64_t n, std::vector<int64_t>& cur, std::vector<std::vector<int64_t>>* out);

// CPython's random.Random (Modules/_randommodule.c, Lib/random.py): MT19937
// seeded by init_by_array over the 32-bit words of |seed|, getrandbits(k) =
// the top k bits of one output, randrange(n) = _randbelow_with_getrandbits,
// random() = 53 bits from two outputs -- bit-exact, so a resampled replay
// draws the decisions the reference draws for the same seed.
class PyRandom {
 public:
  explicit PyRandom(uint64_t seed) {
    uint32_t key[2] = {static_cast<uint32_t>(seed), static_cast<uint32_t>(seed >> 32)};
    init_by_array(key, key[1] ? 2 : 1);
  }
  uint32_t next() {
    if (idx_ >= 624) twist();
    uint32_t y = mt_[idx_++];
    y ^= y >> 11;
    y ^= (y << 7) & 0x9d2c5680u;
    y ^= (y << 15) & 0xefc60000u;
    y ^= y >> 18;
    return y;
  }
  uint32_t getrandbits(int k) { return k <= 0 ? 0u : next() >> (32 - k); }
  int64_t randbelow(int64_t n) {  // n >= 1, n < 2**32
    int k = 0;
    while ((int64_t{1} << k) <= n) ++k;  // n.bit_length()
    int64_t r = getrandbits(k);
    while (r >= n) r = getrandbits(k);
    return r;
  }
  double random() {
    const uint32_t a = next() >> 5, b = next() >> 6;
    return (a * 67108864.0 + b) * (1.0 / 9007199254740992.0);
  }

 private:
  void init_genrand(uint32_t s) {
    mt_[0] = s;
    for (int i = 1; i < 624; ++i) mt_[i] = 1812433253u * (mt_[i - 1] ^ (mt_[i - 1] >> 30)) + static_cast<uint32_t>(i);
    idx_ = 624;
  }
  void init_by_array(const uint32_t* key, int len) {
    init_genrand(19650218u);
    int i = 1, j = 0;
    for (int k = 624 > len ? 624 : len; k; --k) {
      mt_[i] = (mt_[i] ^ ((mt_[i - 1] ^ (mt_[i - 1] >> 30)) * 1664525u)) + key[j] + static_cast<uint32_t>(j);
      ++i;
      ++j;
      if (i >= 624) {
        mt_[0] = mt_[623];
        i = 1;
      }
      if (j >= len) j = 0;
    }
    for (int k = 623; k; --k) {
      mt_[i] = (mt_[i] ^ ((mt_[i - 1] ^ (mt_[i - 1] >> 30)) * 1566083941u)) - static_cast<uint32_t>(i);
      ++i;
      if (i >= 624) {
        mt_[0] = mt_[623];
        i = 1;
      }
    }
    mt_[0] = 0x80000000u;
  }
  void twist() {
    for (int i = 0; i < 624; ++i) {
      const uint32_t y = (mt_[i] & 0x80000000u) | (mt_[(i + 1) % 624] & 0x7fffffffu);
      mt_[i] = mt_[(i + 397) % 624] ^ (y >> 1) ^ ((y & 1u) ? 0x9908b0dfu : 0u);
    }
    idx_ = 0;
  }
  uint32_t mt_[624];
  int idx_ = 624;
};

enum RefKind : uint8_t { RK_BLOCK, RK_LOOP, RK_RV };
enum LocKind : uint8_t { L_ROOT, L_INLINE, L_LOOP };
struct Ref {
  int idx = -1;  // position in the state's handle table
  std::string id;
  RefKind k;
  std::string payload;  // block name / loop var
  bool rv_int = true;   // RV payload ("int", value) or ("loc", token)
  Value ival;           // RV int value (a JSON value: tile factor or categorical candidate)
  LocKind loc = L_ROOT;
  std::string locvar;
  bool alive = true;
  const char* type_name() const { return k == RK_BLOCK ? "BlockRef" : k == RK_LOOP ? "LoopRef" : "RandomVarRef"; }
};

// A resolved instruction argument: a handle, a plain JSON value, or a list.
struct Arg {
  Ref* ref = nullptr;
  const Value* val = nullptr;
  bool is_list = false;
  std::vector<Arg> list;
};
std::string py_type_name(const Arg& a) {
  if (a.ref) return a.ref->type_name();
  if (a.is_list) return "list";
  switch (a.val->t) {
    case Value::Null: return "NoneType";
    case Value::Bool: return "bool";
    case Value::Int: return "int";
    case Value::Float: return "float";
    case Value::Str: return "str";
    case Value::Arr: return "list";
    default: return "dict";
  }
}

int64_t prod(const std::vector<int64_t>& v, size_t from = 0) {
  int64_t p = 1;
  for (size_t i = from; i < v.size(); ++i) p *= v[i];
  return p;
}

// number of ordered n-factorizations of `extent` (len(ordered_factorizations))
int64_t n_factorizations(int64_t extent, int64_t n) {
  static thread_local std::map<std::pair<int64_t, int64_t>, int64_t> memo;
  if (n == 1) return 1;
  auto key = std::make_pair(extent, n);
  auto it = memo.find(key);
  if (it != memo.end()) return it->second;
  int64_t total = 0;
  for (int64_t d = 1; d * d <= extent; ++d) {
    if (extent % d) continue;
    total += n_factorizations(extent / d, n - 1);
    if (d != extent / d) total += n_factorizations(d, n - 1);
  }
  memo[key] = total;
  return total;
}

EP simplify_affine(const EP& e) {
  auto dec = affine_coeffs(e);
  if (!dec) return e;
  const Coeffs& c = dec->first;
  EP expr = (dec->second != 0 || c.empty()) ? mk_int(dec->second) : nullptr;
  for (const auto& kv : c) {  // std::map: sorted(coeffs)
    EP term = kv.second == 1 ? mk_var(kv.first) : mk_bin(E_MUL, mk_var(kv.first), mk_int(kv.second));
    expr = expr ? mk_bin(E_ADD, expr, term) : term;
  }
  return expr;
}

std::optional<int64_t> mixed_radix_width(std::vector<std::pair<int64_t, int64_t>> terms) {
  std::sort(terms.begin(), terms.end());
  int64_t cover = 1;
  for (const auto& t : terms) {
    if (t.first <= 0 || t.first > cover) return std::nullopt;
    cover += t.first * (t.second - 1);
  }
  return cover;
}

struct Access {
  std::vector<EP> idx;
  std::vector<int64_t> tile;
};
using Boxes = std::vector<std::pair<EP, int64_t>>;

class State {
 public:
  Prog prog;
  std::string text;  // recorded (normalized) instructions, serialize_trace lines
  // e0_vars: the loop variables of the workload program, the only names a
  // fresh "x<n>" variable can collide with
  State(Prog p, const std::set<std::string>* e0_vars) : prog(std::move(p)), e0_vars_(e0_vars) {}
  // resample mode (replay(..., mode="resample", seed)): the samplers draw
  // from this generator instead of following the recorded decisions
  std::shared_ptr<PyRandom> rng;

  Ref* ref_at(int i) { return &refs_[static_cast<size_t>(i)]; }
  Ref* new_ref(RefKind k, std::string payload) {
    refs_.emplace_back();
    Ref& r = refs_.back();
    r.idx = static_cast<int>(refs_.size()) - 1;
    r.id = "%" + std::to_string(ref_counter_++);
    r.k = k;
    r.payload = std::move(payload);
    return &r;
  }
  std::string fresh_var() { return "x" + std::to_string(var_counter_++); }

  void set_program(Prog p) {
    auto d = validate_ir(p);
    if (!d.empty()) {
      std::string m = "transformation produced invalid IR: ";
      for (size_t i = 0; i < d.size(); ++i) m += (i ? "; " : "") + d[i];
      sched_err(m);
    }
    prog = std::move(p);
  }
  // split / fuse / reorder / set_kind applied to a valid program can only
  // produce invalid IR through a fresh loop variable that collides with an
  // existing one (every index they write is affine or a floordiv/mod of a
  // fresh variable by a positive constant, every variable they introduce is
  // bound by the loop they create, buffers and blocks are untouched); skip
  // the whole-program validate_ir then -- its verdict is known to be empty
  void set_program_checked_vars(Prog p, const std::vector<std::string>& fresh) {
    for (const auto& v : fresh)
      if (!e0_vars_ || e0_vars_->count(v)) return set_program(std::move(p));
    prog = std::move(p);
  }
  Prog with_root(std::vector<SP> root) const {
    Prog p;
    p.bufs = prog.bufs;
    p.root = std::move(root);
    return p;
  }
  void kill_loops(const std::set<std::string>& vars) {
    for (Ref& r : refs_)
      if (r.k == RK_LOOP && vars.count(r.payload)) r.alive = false;
  }
  void kill_blocks(const std::set<std::string>& names) {
    for (Ref& r : refs_)
      if (r.k == RK_BLOCK && names.count(r.payload)) r.alive = false;
  }

  // -- recording --
  static Value enc(const Arg& a) {
    if (a.ref) return Value::str(a.ref->id);
    if (a.is_list) {
      Value l = Value::arr();
      for (const Arg& x : a.list) l.a.push_back(enc(x));
      return l;
    }
    return *a.val;
  }
  // one line of serialize_trace (src/trace.py:80-86): json.dumps(ins.to_json(),
  // sort_keys=True), keys attrs < decision < inputs < op < outputs
  void record(const char* op, std::vector<Value> inputs, const Value& attrs, const std::vector<Ref*>& outputs,
              const Value* decision = nullptr) {
    std::string& t = text;
    t += "{\"attrs\": ";
    pj::dump(attrs, &t);
    if (decision) {
      t += ", \"decision\": ";
      pj::dump(*decision, &t);
    }
    t += ", \"inputs\": [";
    for (size_t i = 0; i < inputs.size(); ++i) {
      if (i) t += ", ";
      pj::dump(inputs[i], &t);
    }
    t += "], \"op\": ";
    pj::dump_string(op, &t);
    t += ", \"outputs\": [";
    for (size_t i = 0; i < outputs.size(); ++i) {
      if (i) t += ", ";
      pj::dump_string(outputs[i]->id, &t);
    }
    t += "]}\n";
  }

  // -- resolution (src/schedule.py:226-257) --
  std::pair<Path, SP> resolve_loop(const Arg& a) {
    if (!a.ref || a.ref->k == RK_BLOCK) sched_err("expected a loop handle, got " + py_type_name(a));
    Ref* r = a.ref;
    std::string var;
    if (r->k == RK_RV) {
      if (r->rv_int || r->loc != L_LOOP) sched_err(r->id + " is not a loop location");
      var = r->locvar;
    } else {
      var = r->payload;
    }
    auto path = find_loop(prog.root, var);
    if (!r->alive || !path) sched_err("dead handle " + r->id + " (loop " + var + ")");
    return {*path, get_stmt(prog.root, *path)};
  }
  std::pair<Path, SP> resolve_block(const Arg& a) {
    if (!a.ref || a.ref->k != RK_BLOCK) sched_err("expected a block handle, got " + py_type_name(a));
    auto path = find_block(prog.root, a.ref->payload);
    if (!a.ref->alive || !path) sched_err("dead handle " + a.ref->id + " (block " + a.ref->payload + ")");
    return {*path, get_stmt(prog.root, *path)};
  }
  int64_t resolve_factor(const Arg& f) {
    if (f.ref && f.ref->k == RK_RV) {
      if (!f.ref->alive) sched_err("dead handle " + f.ref->id);
      if (!f.ref->rv_int) sched_err(f.ref->id + " is not an integer random variable");
      if (f.ref->ival.t != Value::Int || f.ref->ival.big) defer("non-integer factor value");
      return f.ref->ival.i;
    }
    if (!f.ref && !f.is_list && f.val->t == Value::Int && !f.val->big) return f.val->i;
    if (!f.ref && !f.is_list && f.val->t == Value::Bool) defer("bool factor");
    sched_err("factor must be int or random variable, got " + py_type_name(f));
  }

  // -- analysis primitives --
  std::vector<Ref*> get_blocks() {
    std::vector<Ref*> refs;
    iter_stmts(prog.root, [&](const Path&, const St& s) {
      if (is_block(s)) refs.push_back(new_ref(RK_BLOCK, block_name(s)));
    });
    record("get_blocks", {}, Value::obj(), refs);
    return refs;
  }
  std::vector<Ref*> get_loops(const Arg& block) {
    auto [path, stmt] = resolve_block(block);
    std::vector<Ref*> refs;
    const std::vector<SP>* list = &prog.root;
    for (size_t d = 0; d + 1 < path.size(); ++d) {
      const SP& node = (*list)[path[d]];
      refs.push_back(new_ref(RK_LOOP, node->var));
      list = &node->body;
    }
    record("get_loops", {enc(block)}, Value::obj(), refs);
    return refs;
  }

  // -- transformations --
  std::vector<Ref*> split(const Arg& loop, const Arg& factors) {
    auto [path, node] = resolve_loop(loop);
    if (!factors.is_list) defer("split factors are not a list");
    std::vector<int64_t> vals;
    for (const Arg& f : factors.list) vals.push_back(resolve_factor(f));
    bool bad = vals.empty();
    for (int64_t v : vals) bad |= v < 1;
    if (bad) sched_err("split factors must be positive");
    if (prod(vals) != node->extent)
      sched_err("split of " + node->var + ": factor product " + std::to_string(prod(vals)) + " != extent " +
                std::to_string(node->extent));
    std::vector<std::string> nv;
    for (size_t i = 0; i < vals.size(); ++i) nv.push_back(fresh_var());
    EP recomb;
    for (size_t i = 0; i < nv.size(); ++i) {
      const int64_t inner = prod(vals, i + 1);
      EP term = inner != 1 ? mk_bin(E_MUL, mk_var(nv[i]), mk_int(inner)) : mk_var(nv[i]);
      recomb = recomb ? mk_bin(E_ADD, recomb, term) : term;
    }
    Subst m{{node->var, recomb}};
    std::vector<SP> nest;
    for (const SP& s : node->body) nest.push_back(substitute_stmt(s, m));
    for (size_t i = nv.size(); i-- > 0;) nest = {mk_loop(nv[i], vals[i], "serial", std::move(nest))};
    set_program_checked_vars(with_root(replace_stmt(prog.root, path, nest)), nv);
    kill_loops({node->var});
    std::vector<Ref*> refs;
    for (const auto& v : nv) refs.push_back(new_ref(RK_LOOP, v));
    record("split", {enc(loop), enc(factors)}, Value::obj(), refs);
    return refs;
  }

  std::vector<std::pair<Path, SP>> loop_chain(const std::vector<Arg>& refs) {
    std::vector<std::pair<Path, SP>> r;
    for (const Arg& a : refs) r.push_back(resolve_loop(a));
    std::stable_sort(r.begin(), r.end(), [](const auto& x, const auto& y) { return x.first.size() < y.first.size(); });
    for (size_t i = 0; i + 1 < r.size(); ++i) {
      const Path &p1 = r[i].first, &p2 = r[i + 1].first;
      bool ok = p2.size() == p1.size() + 1 && std::equal(p1.begin(), p1.end(), p2.begin()) &&
                r[i].second->body.size() == 1;
      if (!ok)
        sched_err("loops " + r[i].second->var + " and " + r[i + 1].second->var + " are not adjacent in a perfect nest");
    }
    return r;
  }

  static std::pair<bool, bool> block_var_use(const St& s, const std::string& v) {
    if (s.k == S_COMP) {
      std::set<std::string> store = vars_of(s.idx);
      std::set<std::string> used = vars_of(s.value);
      if (s.init) expr_vars(s.init, &used);
      const bool red = s.init && used.count(v) && !store.count(v);
      return {store.count(v) > 0, red};
    }
    std::set<std::string> store = vars_of(s.ops[0].second), in;
    for (size_t k = 1; k < s.ops.size(); ++k) expr_vars_list(s.ops[k].second, &in);
    return {store.count(v) > 0, in.count(v) && !store.count(v)};
  }
  static void expr_vars_list(const std::vector<EP>& es, std::set<std::string>* out) {
    for (const EP& e : es) expr_vars(e, out);
  }
  static std::vector<const St*> enclosed_blocks(const SP& node) {
    std::vector<const St*> out;
    iter_stmts(std::vector<SP>{node}, [&](const Path&, const St& s) {
      if (is_block(s)) out.push_back(&s);
    });
    return out;
  }
  static const char* loop_role(const SP& node) {
    bool par = true, red = true;
    for (const St* s : enclosed_blocks(node)) {
      auto [in_store, r] = block_var_use(*s, node->var);
      if (r || !in_store) par = false;
      if (!r) red = false;
    }
    return par ? "parallel" : red ? "reduction" : "mixed";
  }

  Ref* fuse(const Arg& loops) {
    if (!loops.is_list) defer("fuse argument is not a list");
    if (loops.list.empty()) sched_err("fuse of an empty loop list");
    auto chain = loop_chain(loops.list);
    std::set<std::string> roles;
    for (const auto& pl : chain) roles.insert(loop_role(pl.second));
    if (roles.size() > 1 || roles.count("mixed")) sched_err("fuse requires all-data-parallel or all-reduction loops");
    if (chain.size() == 1) {
      Ref* r = new_ref(RK_LOOP, chain[0].second->var);
      record("fuse", {enc(loops)}, Value::obj(), {r});
      return r;
    }
    const std::vector<SP>& inner = chain.back().second->body;
    std::vector<int64_t> ext;
    for (const auto& pl : chain) ext.push_back(pl.second->extent);
    const std::string fv = fresh_var();
    Subst m;
    for (size_t i = 0; i < chain.size(); ++i) {
      const int64_t ip = prod(ext, i + 1);
      EP e = mk_var(fv);
      if (ip != 1) e = mk_bin(E_FDIV, e, mk_int(ip));
      if (i > 0) e = mk_bin(E_MOD, e, mk_int(chain[i].second->extent));
      m[chain[i].second->var] = e;
    }
    std::vector<SP> body;
    for (const SP& s : inner) body.push_back(substitute_stmt(s, m));
    SP fused = mk_loop(fv, prod(ext), "serial", std::move(body));
    set_program_checked_vars(with_root(replace_stmt(prog.root, chain[0].first, {fused})), {fv});
    std::set<std::string> dead;
    for (const auto& pl : chain) dead.insert(pl.second->var);
    kill_loops(dead);
    Ref* r = new_ref(RK_LOOP, fv);
    record("fuse", {enc(loops)}, Value::obj(), {r});
    return r;
  }

  void reorder(const Arg& loops) {
    if (!loops.is_list) defer("reorder argument is not a list");
    if (loops.list.empty()) sched_err("reorder of an empty loop list");
    auto chain = loop_chain(loops.list);
    std::vector<std::pair<Path, SP>> resolved;
    for (const Arg& a : loops.list) resolved.push_back(resolve_loop(a));
    std::vector<SP> nest = chain.back().second->body;
    for (size_t i = resolved.size(); i-- > 0;) {
      const SP& n = resolved[i].second;
      nest = {mk_loop(n->var, n->extent, n->kind, std::move(nest))};
    }
    set_program_checked_vars(with_root(replace_stmt(prog.root, chain[0].first, nest)), {});
    record("reorder", {enc(loops)}, Value::obj(), {});
  }

  void set_kind(const Arg& loop, const char* kind, const char* op) {
    auto [path, node] = resolve_loop(loop);
    auto n = std::make_shared<St>(*node);
    n->kind = kind;
    set_program_checked_vars(with_root(replace_stmt(prog.root, path, {n})), {});
    record(op, {enc(loop)}, Value::obj(), {});
  }
  void require_data_parallel(const SP& node, const char* what) {
    for (const St* s : enclosed_blocks(node)) {
      auto [in_store, red] = block_var_use(*s, node->var);
      if (red)
        sched_err(std::string(what) + ": reduction-carried dependence on " + node->var + " in block " + block_name(*s));
      if (!in_store)
        sched_err(std::string(what) + ": loop var " + node->var + " is absent from the store index of block " +
                  block_name(*s));
    }
  }
  void parallelize(const Arg& loop) {
    auto pn = resolve_loop(loop);
    require_data_parallel(pn.second, "parallelize");
    set_kind(loop, "parallel", "parallelize");
  }
  void vectorize(const Arg& loop) {
    auto pn = resolve_loop(loop);
    require_data_parallel(pn.second, "vectorize");
    bool nested = false;
    iter_stmts(pn.second->body, [&](const Path&, const St& s) { nested |= s.k == S_LOOP; });
    if (nested) sched_err("vectorize: loop " + pn.second->var + " is not innermost in its nest");
    set_kind(loop, "vectorized", "vectorize");
  }
  void unroll(const Arg& loop) {
    auto pn = resolve_loop(loop);
    if (pn.second->extent > 64)
      sched_err("unroll: extent " + std::to_string(pn.second->extent) + " exceeds 64");
    set_kind(loop, "unrolled", "unroll");
  }

  // -- producer/consumer analysis (src/schedule.py:432-604) --
  std::optional<std::string> writer_of(const std::string& buf) const {
    std::optional<std::string> w;
    iter_stmts(prog.root, [&](const Path&, const St& s) {
      if (w) return;
      if (s.k == S_COMP && s.buffer == buf) w = s.name;
      else if (s.k == S_INTR && !s.ops.empty() && s.ops[0].first == buf) w = s.block;
    });
    return w;
  }
  std::vector<std::string> readers_of(const std::string& buf) const {
    std::vector<std::string> out;
    iter_stmts(prog.root, [&](const Path&, const St& s) {
      std::optional<std::string> name;
      if (s.k == S_COMP) {
        if (s.buffer != buf) {
          std::vector<const Ex*> lds;
          collect_loads(s.value, &lds);
          collect_loads(s.init, &lds);
          collect_loads(s.epi, &lds);
          for (const Ex* l : lds)
            if (l->s == buf) name = s.name;
        }
      } else if (s.k == S_INTR) {
        bool reads = false;
        for (size_t k = 1; k < s.ops.size(); ++k) reads |= s.ops[k].first == buf;
        if (s.ops[0].first != buf && reads) name = s.block;
      }
      if (name && std::find(out.begin(), out.end(), *name) == out.end()) out.push_back(*name);
    });
    return out;
  }
  bool is_elementwise(const St& s) const {
    if (s.k != S_COMP || s.init || s.epi) return false;
    std::vector<std::string> names;
    for (const EP& i : s.idx) {
      if (i->k != E_VAR) return false;
      names.push_back(i->s);
    }
    std::set<std::string> ns(names.begin(), names.end());
    if (ns.size() != names.size()) return false;
    auto path = find_block(prog.root, s.name);
    std::set<std::string> lv;
    for (const auto& pl : enclosing_loops(prog.root, *path)) lv.insert(pl.second->var);
    return ns == lv;
  }
  const St& block_stmt(const std::string& name) const { return *get_stmt(prog.root, *find_block(prog.root, name)); }
  static const std::string& out_buffer(const St& s) { return s.k == S_COMP ? s.buffer : s.ops[0].first; }

  std::optional<std::pair<std::string, bool>> counterpart(const St& b) const {  // (name, at_producer)
    std::vector<std::string> produced;
    std::vector<const Ex*> lds;
    collect_loads(b.value, &lds);
    for (const Ex* l : lds) {
      auto w = writer_of(l->s);
      if (w && *w != b.name && std::find(produced.begin(), produced.end(), *w) == produced.end())
        produced.push_back(*w);
    }
    if (produced.size() == 1) {
      const St& ps = block_stmt(produced[0]);
      if (readers_of(out_buffer(ps)) == std::vector<std::string>{b.name}) return std::make_pair(produced[0], true);
    }
    auto readers = readers_of(b.buffer);
    if (readers.size() == 1) return std::make_pair(readers[0], false);
    return std::nullopt;
  }

  static std::vector<Access> access_terms(const St& s, const std::string& buf, bool writes) {
    std::vector<Access> out;
    if (s.k == S_COMP) {
      if (writes) {
        if (s.buffer == buf) out.push_back({s.idx, std::vector<int64_t>(s.idx.size(), 1)});
      } else {
        for (const EP& e : {s.value, s.init, s.epi}) {
          std::vector<const Ex*> lds;
          collect_loads(e, &lds);
          for (const Ex* l : lds)
            if (l->s == buf) out.push_back({l->a, std::vector<int64_t>(l->a.size(), 1)});
        }
      }
    } else if (s.k == S_INTR) {
      const IntrInfo* info = intrinsic(s.name);
      if (!info) defer("unknown intrinsic in program");
      const size_t lo = writes ? 0 : 1, hi = writes ? std::min<size_t>(1, s.ops.size()) : s.ops.size();
      for (size_t k = lo; k < hi; ++k)
        if (s.ops[k].first == buf)
          out.push_back({s.ops[k].second, std::vector<int64_t>(s.ops[k].second.size(), info->tile[0])});
    }
    return out;
  }

  static std::optional<Boxes> region_boxes(const std::vector<Access>& acc, const std::set<std::string>& outer,
                                           const std::map<std::string, int64_t>& inner) {
    const size_t ndim = acc[0].idx.size();
    Boxes boxes;
    for (size_t d = 0; d < ndim; ++d) {
      struct Entry {
        Coeffs outer_part;
        int64_t c0, width;
      };
      std::vector<Entry> entries;
      for (const Access& a : acc) {
        if (d >= a.idx.size()) defer("ragged access ranks");
        auto dec = affine_coeffs(a.idx[d]);
        if (!dec) return std::nullopt;
        std::vector<std::pair<int64_t, int64_t>> terms;
        for (const auto& kv : dec->first) {
          auto it = inner.find(kv.first);
          if (it != inner.end()) terms.push_back({kv.second, it->second});
        }
        for (const auto& kv : dec->first)
          if (!inner.count(kv.first) && !outer.count(kv.first)) return std::nullopt;
        if (a.tile[d] > 1) terms.push_back({1, a.tile[d]});
        int64_t width = 1;
        if (!terms.empty()) {
          auto w = mixed_radix_width(terms);
          if (!w) return std::nullopt;
          width = *w;
        }
        Coeffs op;
        for (const auto& kv : dec->first)
          if (outer.count(kv.first)) op[kv.first] = kv.second;
        entries.push_back({std::move(op), dec->second, width});
      }
      for (const Entry& e : entries)
        if (e.outer_part != entries[0].outer_part) return std::nullopt;
      int64_t lo = entries[0].c0, hi = entries[0].c0 + entries[0].width;
      for (const Entry& e : entries) {
        lo = std::min(lo, e.c0);
        hi = std::max(hi, e.c0 + e.width);
      }
      EP expr = mk_int(lo);
      for (const auto& kv : entries[0].outer_part) {
        EP term = kv.second == 1 ? mk_var(kv.first) : mk_bin(E_MUL, mk_var(kv.first), mk_int(kv.second));
        expr = (expr->k == E_INT && expr->v == 0) ? term : mk_bin(E_ADD, expr, term);
      }
      boxes.push_back({expr, hi - lo});
    }
    return boxes;
  }

  static std::vector<std::string> reduction_vars(const St& s, const std::vector<std::string>& loop_vars) {
    std::vector<std::string> out;
    if (s.k == S_COMP) {
      if (!s.init) return out;
      std::set<std::string> store = vars_of(s.idx), used = vars_of(s.value);
      expr_vars(s.init, &used);
      for (const auto& v : loop_vars)
        if (used.count(v) && !store.count(v)) out.push_back(v);
    } else {
      std::set<std::string> ov = vars_of(s.ops[0].second), iv;
      for (size_t k = 1; k < s.ops.size(); ++k) expr_vars_list(s.ops[k].second, &iv);
      for (const auto& v : loop_vars)
        if (iv.count(v) && !ov.count(v)) out.push_back(v);
    }
    return out;
  }

  std::optional<std::pair<Boxes, std::vector<std::string>>> attach_analysis(const St& b, const std::string& cp_name,
                                                                             bool at_producer, size_t depth) const {
    const Path cp_path = *find_block(prog.root, cp_name);
    const St& cp = *get_stmt(prog.root, cp_path);
    auto cp_loops = enclosing_loops(prog.root, cp_path);
    if (depth >= cp_loops.size()) return std::nullopt;
    std::set<std::string> outer;
    for (size_t i = 0; i <= depth; ++i) outer.insert(cp_loops[i].second->var);
    std::map<std::string, int64_t> inner;
    for (size_t i = depth + 1; i < cp_loops.size(); ++i) inner[cp_loops[i].second->var] = cp_loops[i].second->extent;
    std::vector<std::string> cp_vars;
    for (const auto& pl : cp_loops) cp_vars.push_back(pl.second->var);
    if (at_producer) {
      for (const auto& v : reduction_vars(cp, cp_vars))
        if (outer.count(v)) return std::nullopt;
      const std::string& pbuf = out_buffer(cp);
      auto reads = access_terms(b, pbuf, false);
      if (reads.size() != 1) return std::nullopt;
      const auto& ridx = reads[0].idx;
      std::vector<std::string> names;
      for (const EP& i : ridx) {
        if (i->k != E_VAR) return std::nullopt;
        names.push_back(i->s);
      }
      if (std::set<std::string>(names.begin(), names.end()).size() != names.size()) return std::nullopt;
      std::map<std::string, int64_t> ext;
      for (const auto& pl : enclosing_loops(prog.root, *find_block(prog.root, b.name)))
        ext[pl.second->var] = pl.second->extent;
      const Buf* pb = prog.buffer(pbuf);
      if (!pb) defer("unknown producer buffer");
      for (size_t d = 0; d < names.size(); ++d) {
        auto it = ext.find(names[d]);
        if (d >= pb->shape.size()) defer("rank mismatch");
        if (it == ext.end() || it->second != pb->shape[d]) return std::nullopt;
      }
      auto writes = access_terms(cp, pbuf, true);
      if (writes.empty()) defer("producer without a write");
      auto boxes = region_boxes(writes, outer, inner);
      if (!boxes) return std::nullopt;
      return std::make_pair(std::move(*boxes), names);
    }
    auto reads = access_terms(cp, b.buffer, false);
    if (reads.empty()) return std::nullopt;
    auto boxes = region_boxes(reads, outer, inner);
    if (!boxes) return std::nullopt;
    std::vector<std::string> store;
    for (const EP& i : b.idx) store.push_back(i->s);
    return std::make_pair(std::move(*boxes), store);
  }

  struct AttachCand {
    std::string cp_name;
    bool at_producer;
    std::vector<std::string> loops;
  };
  std::optional<AttachCand> attach_candidates(const St& b) const {
    auto cp = counterpart(b);
    if (!cp) return std::nullopt;
    auto cp_loops = enclosing_loops(prog.root, *find_block(prog.root, cp->first));
    AttachCand out{cp->first, cp->second, {}};
    for (size_t d = 0; d < cp_loops.size(); ++d)
      if (attach_analysis(b, cp->first, cp->second, d)) out.loops.push_back(cp_loops[d].second->var);
    return out;
  }

  Path exclusive_nest_path(Path path) const {
    while (path.size() > 1) {
      Path parent(path.begin(), path.end() - 1);
      if (get_stmt(prog.root, parent)->body.size() != 1) return path;
      path = parent;
    }
    return path;
  }

  void compute_at(const Arg& block, const Arg* loop) {
    const bool root = !loop || (!loop->ref && !loop->is_list &&
                                ((loop->val->t == Value::Str && loop->val->s == "root") || loop->val->t == Value::Null)) ||
                      (loop->ref && loop->ref->k == RK_RV && !loop->ref->rv_int && loop->ref->loc == L_ROOT);
    if (root) {
      resolve_block(block);
      Value attrs = Value::obj();
      attrs.put("location", Value::str("root"));
      record("compute_at", {enc(block)}, std::move(attrs), {});
      return;
    }
    auto [bpath, bs] = resolve_block(block);
    auto [lpath, lnode] = resolve_loop(*loop);
    if (!is_elementwise(*bs)) sched_err("compute_at: block " + block_name(*bs) + " is not elementwise");
    auto cp = counterpart(*bs);
    if (!cp) sched_err("compute_at: block " + bs->name + " has no unique producer/consumer counterpart");
    const std::string cp_name = cp->first;
    const bool at_producer = cp->second;
    auto cp_loops = enclosing_loops(prog.root, *find_block(prog.root, cp_name));
    std::optional<size_t> depth;
    for (size_t i = 0; i < cp_loops.size(); ++i)
      if (cp_loops[i].second->var == lnode->var) {
        depth = i;
        break;
      }
    if (!depth) sched_err("compute_at: loop " + lnode->var + " does not belong to the nest of " + cp_name);
    auto an = attach_analysis(*bs, cp_name, at_producer, *depth);
    if (!an) sched_err("compute_at: dependence violation attaching " + bs->name + " at " + lnode->var);
    const Boxes& boxes = an->first;
    const auto& dim_vars = an->second;
    Subst mapping;
    std::vector<std::pair<std::string, int64_t>> to_make;
    for (size_t d = 0; d < boxes.size(); ++d) {
      if (d >= dim_vars.size()) defer("box/dim mismatch");
      const std::string& v = dim_vars[d];
      if (boxes[d].second == 1) {
        mapping[v] = simplify_affine(boxes[d].first);
      } else {
        std::string nv = fresh_var();
        to_make.push_back({nv, boxes[d].second});
        mapping[v] = simplify_affine(mk_bin(E_ADD, boxes[d].first, mk_var(nv)));
      }
    }
    SP new_stmt = substitute_stmt(bs, mapping);
    std::vector<SP> nest{new_stmt};
    for (size_t i = to_make.size(); i-- > 0;) nest = {mk_loop(to_make[i].first, to_make[i].second, "serial", nest)};
    const Path old_nest = exclusive_nest_path(bpath);
    std::set<std::string> old_vars;
    iter_stmts(std::vector<SP>{get_stmt(prog.root, old_nest)}, [&](const Path&, const St& s) {
      if (s.k == S_LOOP) old_vars.insert(s.var);
    });
    std::vector<SP> r = replace_stmt(prog.root, old_nest, {});
    auto cpp = find_block(r, cp_name);
    if (!cpp) defer("counterpart removed");
    std::optional<Path> attach_path;
    for (const auto& pl : enclosing_loops(r, *cpp))
      if (pl.second->var == lnode->var) attach_path = pl.first;
    if (!attach_path) defer("attach loop removed");
    const SP& attach = get_stmt(r, *attach_path);
    const int child = (*cpp)[attach_path->size()];
    std::vector<SP> body;
    const int cut = at_producer ? child + 1 : child;
    body.insert(body.end(), attach->body.begin(), attach->body.begin() + cut);
    body.insert(body.end(), nest.begin(), nest.end());
    body.insert(body.end(), attach->body.begin() + cut, attach->body.end());
    r = replace_stmt(r, *attach_path, {with_body(*attach, std::move(body))});
    set_program(with_root(std::move(r)));
    kill_loops(old_vars);
    record("compute_at", {enc(block), enc(*loop)}, Value::obj(), {});
  }

  // -- inline (src/schedule.py:739-857) --
  std::optional<bool> inline_mode(const St& s) const {  // true forward, false reverse
    if (!is_elementwise(s)) return std::nullopt;
    const Buf* buf = prog.buffer(s.buffer);
    if (!buf) defer("unknown buffer");
    auto readers = readers_of(s.buffer);
    if (buf->role == "intermediate" && readers.size() == 1) {
      if (block_stmt(readers[0]).k == S_COMP) return true;
    }
    std::vector<std::pair<std::string, std::string>> produced;
    std::vector<const Ex*> lds;
    collect_loads(s.value, &lds);
    for (const Ex* l : lds) {
      auto w = writer_of(l->s);
      if (w && *w != s.name) {
        auto key = std::make_pair(*w, l->s);
        if (std::find(produced.begin(), produced.end(), key) == produced.end()) produced.push_back(key);
      }
    }
    if (produced.size() == 1) {
      const std::string& pname = produced[0].first;
      const std::string& pbuf = produced[0].second;
      const St& ps = block_stmt(pname);
      const Buf* pb = prog.buffer(pbuf);
      if (!pb) defer("unknown buffer");
      if (ps.k == S_COMP && pb->role == "intermediate" && readers_of(pbuf) == std::vector<std::string>{s.name}) {
        std::vector<const Ex*> pl;
        for (const Ex* l : lds)
          if (l->s == pbuf) pl.push_back(l);
        if (pl.size() == 1) {
          std::vector<std::string> li, si;
          bool all_var = true;
          for (const EP& i : pl[0]->a) {
            all_var &= i->k == E_VAR;
            if (i->k == E_VAR) li.push_back(i->s);
          }
          for (const EP& i : s.idx) si.push_back(i->s);
          std::set<std::string> ls(li.begin(), li.end()), ss(si.begin(), si.end());
          if (all_var && ls == ss && ls.size() == pl[0]->a.size()) {
            if (ps.epi && li != si) return std::nullopt;
            return false;
          }
        }
      }
    }
    return std::nullopt;
  }

  static EP map_loads(const EP& e, const std::string& buf, const std::function<EP(const std::vector<EP>&)>& fn) {
    if (!e || e->k == E_INT || e->k == E_VAR) return e;
    if (e->k == E_LOAD) {
      std::vector<EP> idx;
      for (const EP& i : e->a) idx.push_back(map_loads(i, buf, fn));
      if (e->s == buf) return fn(idx);
      return mk_load(e->s, std::move(idx));
    }
    auto n = std::make_shared<Ex>(*e);
    for (EP& c : n->a) c = map_loads(c, buf, fn);
    return n;
  }

  void inline_block(const Arg& block) {
    auto [bpath, bs] = resolve_block(block);
    if (bs->k != S_COMP) sched_err("inline: tensorized blocks cannot be inlined");
    auto mode = inline_mode(*bs);
    if (!mode)
      sched_err("inline: block " + block_name(*bs) +
                " is not inlinable (must be elementwise with a unique producer or consumer)");
    if (*mode) inline_forward(bpath, *bs);
    else inline_reverse(bpath, *bs);
    kill_blocks({bs->name});
    record("inline", {enc(block)}, Value::obj(), {});
  }

  std::set<std::string> loop_vars_under(const Path& p) const {
    std::set<std::string> out;
    iter_stmts(std::vector<SP>{get_stmt(prog.root, p)}, [&](const Path&, const St& s) {
      if (s.k == S_LOOP) out.insert(s.var);
    });
    return out;
  }

  void inline_forward(const Path& bpath, const St& b) {
    const std::string consumer = readers_of(b.buffer)[0];
    std::vector<std::string> store;
    for (const EP& i : b.idx) store.push_back(i->s);
    auto splice = [&](const std::vector<EP>& idx) {
      Subst m;
      for (size_t d = 0; d < store.size() && d < idx.size(); ++d) m[store[d]] = idx[d];
      if (idx.size() < store.size()) defer("rank mismatch in forward inline");
      return substitute(b.value, m);
    };
    const Path cpath = *find_block(prog.root, consumer);
    const SP& cs = get_stmt(prog.root, cpath);
    auto nc = std::make_shared<St>(*cs);
    nc->value = map_loads(cs->value, b.buffer, splice);
    nc->init = map_loads(cs->init, b.buffer, splice);
    nc->epi = map_loads(cs->epi, b.buffer, splice);
    const Path nest = exclusive_nest_path(bpath);
    const std::set<std::string> old_vars = loop_vars_under(nest);
    std::vector<SP> r = replace_stmt(prog.root, cpath, {nc});
    r = replace_stmt(r, nest, {});
    Prog p;
    for (const Buf& x : prog.bufs)
      if (x.name != b.buffer) p.bufs.push_back(x);
    p.root = std::move(r);
    set_program(std::move(p));
    kill_loops(old_vars);
  }

  void inline_reverse(const Path& bpath, const St& b) {
    std::vector<const Ex*> lds;
    collect_loads(b.value, &lds);
    const Ex* pload = nullptr;
    for (const Ex* l : lds) {
      auto w = writer_of(l->s);
      if (w && *w != b.name) {
        pload = l;
        break;
      }
    }
    if (!pload) defer("no producer load");
    const std::string pbuf = pload->s;
    const std::string pname = *writer_of(pbuf);
    const Path ppath = *find_block(prog.root, pname);
    const SP& ps = get_stmt(prog.root, ppath);
    std::vector<std::string> g;
    for (const EP& i : pload->a) g.push_back(i->s);
    std::vector<EP> new_idx;
    for (const EP& i : b.idx) {
      auto it = std::find(g.begin(), g.end(), i->s);
      if (it == g.end() || static_cast<size_t>(it - g.begin()) >= ps->idx.size()) defer("index permutation");
      new_idx.push_back(ps->idx[static_cast<size_t>(it - g.begin())]);
    }
    Subst var_map;
    for (size_t d = 0; d < g.size(); ++d) {
      if (d >= ps->idx.size()) defer("rank mismatch");
      var_map[g[d]] = ps->idx[d];
    }
    auto as_producer_expr = [&](const EP& repl) {
      EP e = substitute(b.value, var_map);
      return map_loads(e, pbuf, [&](const std::vector<EP>&) { return repl; });
    };
    auto np = std::make_shared<St>(*ps);
    np->buffer = b.buffer;
    np->idx = new_idx;
    if (!ps->init) {
      np->value = as_producer_expr(ps->value);
    } else {
      EP composed = ps->epi ? as_producer_expr(rename_loads(ps->epi, pbuf, b.buffer))
                            : as_producer_expr(mk_load(b.buffer, new_idx));
      np->value = rename_loads(ps->value, pbuf, b.buffer);
      np->init = rename_loads(ps->init, pbuf, b.buffer);
      np->epi = composed;
    }
    const Path nest = exclusive_nest_path(bpath);
    const std::set<std::string> old_vars = loop_vars_under(nest);
    std::vector<SP> r = replace_stmt(prog.root, ppath, {np});
    r = replace_stmt(r, nest, {});
    Prog p;
    for (const Buf& x : prog.bufs)
      if (x.name != pbuf) p.bufs.push_back(x);
    p.root = std::move(r);
    set_program(std::move(p));
    kill_loops(old_vars);
  }

  // -- tensorize (src/schedule.py:861-932) --
  void tensorize(const Arg& loop, const Value* name) {
    if (!name || name->t != Value::Str) defer("intrinsic name");
    const IntrInfo* info = intrinsic(name->s);
    if (!info) sched_err("unknown intrinsic " + pj::py_repr(name->s));
    auto [path, node] = resolve_loop(loop);
    std::vector<SP> nest;
    SP cur = node;
    for (int level = 0; level < 3; ++level) {
      if (cur->k != S_LOOP)
        sched_err(std::string("tensorize: expected a 3-deep loop nest, found a ") +
                  (cur->k == S_COMP ? "Compute" : "Intrinsic") + " at level " + std::to_string(level));
      if (cur->extent != info->tile[level])
        sched_err("tensorize: loop " + cur->var + " has extent " + std::to_string(cur->extent) + ", expected " +
                  std::to_string(info->tile[level]));
      if (cur->body.size() != 1) sched_err("tensorize: loop " + cur->var + " must have a single statement body");
      nest.push_back(cur);
      cur = cur->body[0];
    }
    if (cur->k != S_COMP) sched_err("tensorize: innermost statement must be a compute");
    if (!cur->init) sched_err("tensorize: expected a reduction compute (with init)");
    if (cur->epi) sched_err("tensorize: compute with an epilogue cannot be tensorized");
    const std::string av = nest[0]->var, bv = nest[1]->var, cv = nest[2]->var;
    const std::string tile_vars[3] = {av, bv, cv};
    {
      std::set<std::string> iv = vars_of(cur->init);
      for (const auto& v : tile_vars)
        if (iv.count(v)) sched_err("tensorize: init must not depend on the tile loops");
    }
    const EP& val = cur->value;
    if (!(val->k == E_MUL && val->a[0]->k == E_LOAD && val->a[1]->k == E_LOAD))
      sched_err("tensorize: body must be a product of two loads");
    auto coeff_pattern = [&](const EP& e, const std::string* wanted) {
      auto dec = affine_coeffs(e);
      if (!dec) sched_err("tensorize: non-affine index in the tile body");
      for (const auto& v : tile_vars) {
        const int64_t want = (wanted && v == *wanted) ? 1 : 0;
        auto it = dec->first.find(v);
        const int64_t have = it == dec->first.end() ? 0 : it->second;
        if (have != want)
          sched_err("tensorize: index " + expr_str(e) + " must have coefficient " + std::to_string(want) + " on " + v);
      }
      Subst z;
      for (const auto& v : tile_vars) z[v] = mk_int(0);
      return simplify_affine(substitute(e, z));
    };
    if (cur->idx.size() != 2) sched_err("tensorize: output must be 2-dimensional");
    std::vector<EP> c_base{coeff_pattern(cur->idx[0], &av), coeff_pattern(cur->idx[1], &bv)};
    const Ex* loads[2] = {val->a[0].get(), val->a[1].get()};
    const EP lptr[2] = {val->a[0], val->a[1]};
    for (const Ex* l : loads)
      if (l->a.size() != 2) sched_err("tensorize: operands must be 2-dimensional loads");
    int ai = -1;
    for (int k = 0; k < 2 && ai < 0; ++k)
      if (vars_of(lptr[k]).count(av)) ai = k;
    if (ai < 0) sched_err("tensorize: could not match operand loads to the output row index");
    // b_load = next(l for l in loads if l is not a_load): identity, not equality
    const int bi = ai == 0 ? 1 : 0;
    const Ex* al = loads[ai];
    const Ex* bl = loads[bi];
    std::vector<EP> a_base{coeff_pattern(al->a[0], &av), coeff_pattern(al->a[1], &cv)};
    std::vector<EP> b_base{coeff_pattern(bl->a[0], &cv), coeff_pattern(bl->a[1], &bv)};
    auto ns = std::make_shared<St>();
    ns->k = S_INTR;
    ns->name = info->name;
    ns->block = cur->name;
    ns->ops = {{cur->buffer, c_base}, {al->s, a_base}, {bl->s, b_base}};
    ns->init = cur->init;
    set_program(with_root(replace_stmt(prog.root, path, {ns})));
    kill_loops({av, bv, cv});
    Value attrs = Value::obj();
    attrs.put("intrinsic", Value::str(name->s));
    record("tensorize", {enc(loop)}, std::move(attrs), {});
  }

  // -- samplers in decision-following mode (src/schedule.py:936-1018) --
  std::vector<Ref*> sample_perfect_tile(const Arg& loop, const Value* nval, const Value* decision) {
    if (!nval || nval->t != Value::Int || nval->big) defer("sample_perfect_tile n");
    const int64_t n = nval->i;
    if (n < 1) sched_err("sample_perfect_tile: n must be >= 1");
    auto [path, node] = resolve_loop(loop);
    std::vector<int64_t> tile;
    if (rng) {  // domain[_draw_index(len(domain))], the lexicographic domain of ordered_factorizations
      if (n > 8 || node->extent < 1) defer("tile domain");
      std::vector<std::vector<int64_t>> dom;
      std::vector<int64_t> cur;
      factorizations(node->extent, n, cur, &dom);
      tile = dom[static_cast<size_t>(rng->randbelow(static_cast<int64_t>(dom.size())))];
    } else {
      if (!decision || decision->t != Value::Arr) defer("tile decision");
      for (const Value& x : decision->a) {
        if (x.t != Value::Int || x.big) defer("non-integer tile decision");
        tile.push_back(x.i);
      }
    }
    bool bad = static_cast<int64_t>(tile.size()) != n;
    for (int64_t f : tile) bad |= f < 1;
    if (bad || prod(tile) != node->extent)
      sched_err("sample_perfect_tile: decision " + py_int_list(tile) + " is not a perfect " + std::to_string(n) +
                "-way factorization of " + std::to_string(node->extent));
    const int64_t size = n_factorizations(node->extent, n);
    std::vector<Ref*> refs;
    for (int64_t f : tile) {
      Ref* r = new_ref(RK_RV, "");
      r->rv_int = true;
      r->ival = Value::integer(f);
      refs.push_back(r);
    }
    Value attrs = Value::obj();
    attrs.put("n", *nval);
    attrs.put("extent", Value::integer(node->extent));
    Value dec = Value::obj();
    Value tl = Value::arr();
    for (int64_t f : tile) tl.a.push_back(Value::integer(f));
    dec.put("tile", std::move(tl));
    dec.put("size", Value::integer(size));
    record("sample_perfect_tile", {enc(loop)}, std::move(attrs), refs, &dec);
    return refs;
  }

  Ref* sample_categorical(const Value* cands, const Value* probs, const Value* decision) {
    if (!cands || !probs || cands->t != Value::Arr || probs->t != Value::Arr) defer("categorical attrs");
    if (cands->a.size() != probs->a.size()) sched_err("sample_categorical: length mismatch");
    std::vector<double> w;
    for (const Value& p : probs->a) {
      if (p.t == Value::Float) w.push_back(p.d);
      else if (p.t == Value::Int && !p.big) w.push_back(static_cast<double>(p.i));
      else defer("non-numeric weight");
    }
    for (double x : w)
      if (x < 0) sched_err("sample_categorical: negative weight");
    double total = 0;  // float(sum(probs)): Python sums left to right from int 0
    for (double x : w) total += x;
    if (!(total > 0)) sched_err("sample_categorical: all-zero weights");
    int64_t idx;
    if (rng) {  // _draw_index with weights (src/schedule.py:174-186)
      const double r = rng->random() * total;
      double acc = 0.0;
      idx = static_cast<int64_t>(w.size()) - 1;
      for (size_t i = 0; i < w.size(); ++i) {
        acc += w[i];
        if (r < acc) {
          idx = static_cast<int64_t>(i);
          break;
        }
      }
    } else {
      if (!decision || decision->t != Value::Int || decision->big) defer("categorical decision");
      idx = decision->i;
    }
    if (!(0 <= idx && idx < static_cast<int64_t>(cands->a.size())) || w[static_cast<size_t>(idx)] <= 0)
      sched_err("sample_categorical: decision " + std::to_string(idx) + " out of domain");
    Ref* r = new_ref(RK_RV, "");
    r->rv_int = true;
    r->ival = cands->a[static_cast<size_t>(idx)];
    Value attrs = Value::obj();
    attrs.put("candidates", *cands);
    Value pw = Value::arr();
    for (double x : w) pw.a.push_back(Value::real(x));
    attrs.put("probs", std::move(pw));
    Value dec = Value::obj();
    dec.put("index", Value::integer(idx));
    dec.put("prob", Value::real(w[static_cast<size_t>(idx)] / total));
    dec.put("size", Value::integer(static_cast<int64_t>(cands->a.size())));
    record("sample_categorical", {}, std::move(attrs), {r}, &dec);
    return r;
  }

  Ref* sample_compute_location(const Arg& block, const Value* decision) {
    auto [bpath, bs] = resolve_block(block);
    if (bs->k != S_COMP || !is_elementwise(*bs))
      sched_err("sample_compute_location: block " + block_name(*bs) + " is not eligible");
    auto cand = attach_candidates(*bs);
    if (!cand) sched_err("sample_compute_location: block " + bs->name + " has no counterpart");
    const bool can_inline = inline_mode(*bs).has_value();
    const int64_t size = 1 + (can_inline ? 1 : 0) + static_cast<int64_t>(cand->loops.size());
    int64_t idx;
    if (rng) {
      idx = rng->randbelow(size);
    } else {
      if (!decision || decision->t != Value::Int || decision->big) defer("location decision");
      idx = decision->i;
    }
    if (!(0 <= idx && idx < size))
      sched_err("sample_compute_location: decision " + std::to_string(idx) + " outside domain of size " +
                std::to_string(size));
    Ref* r = new_ref(RK_RV, "");
    r->rv_int = false;
    if (idx == 0) {
      r->loc = L_ROOT;
    } else if (can_inline && idx == 1) {
      r->loc = L_INLINE;
    } else {
      r->loc = L_LOOP;
      r->locvar = cand->loops[static_cast<size_t>(idx - 1 - (can_inline ? 1 : 0))];
    }
    Value dec = Value::obj();
    dec.put("index", Value::integer(idx));
    dec.put("size", Value::integer(size));
    record("sample_compute_location", {enc(block)}, Value::obj(), {r}, &dec);
    return r;
  }

 private:
  const std::set<std::string>* e0_vars_ = nullptr;
  std::deque<Ref> refs_;
  int64_t ref_counter_ = 0;
  int64_t var_counter_ = 0;
};

// ---------------------------------------------------------------------------
// replay / validate_trace (src/trace.py:163-265)
// ---------------------------------------------------------------------------

struct ReplayErr {  // ReplayError(index, reason)
  int index;
  std::string reason;
};

struct Outcome {
  int status = LS_REPLAY_DEFER;
  int index = -1;
  uint64_t hash = 0;
  std::string program, trace, reason;
};

#ifdef LSB_REPLAY_PROFILE
std::map<std::string, double> g_prof;
#endif
struct Workload {
  Prog e0;
  std::string text;  // e0 as serialized
  uint64_t hash = 0;
  std::set<std::string> loop_vars;  // of e0
  uint64_t serial = 0;              // identity for the per-thread copies
};

// Every state shares e0's nodes; replaying on several host threads at once
// would make all of them bump the same shared_ptr reference counts (one
// contended cache line per node -- measured: no speed-up at 8 threads), so
// each thread replays from its own deep copy of e0.
const Prog& local_e0(const Workload& w) {
  thread_local std::unordered_map<uint64_t, Prog> copies;
  auto it = copies.find(w.serial);
  if (it != copies.end()) return it->second;
  if (copies.size() > 64) copies.clear();
  Prog p;
  program_from(w.text, &p);
  return copies.emplace(w.serial, std::move(p)).first->second;
}

// replay's `env` (src/trace.py:179-183): trace id -> handle of this state,
// by index so a copied state (a neighbour's prefix snapshot) keeps it valid
struct Env {
  std::vector<int> num;                      // "%<k>" -> handle index, -1 unbound
  std::unordered_map<std::string, int> other;
  static int numeric(const std::string& id) {
    if (id.size() < 2 || id.size() > 9 || id[0] != '%') return -1;
    int v = 0;
    for (size_t i = 1; i < id.size(); ++i) {
      if (id[i] < '0' || id[i] > '9') return -1;
      v = v * 10 + (id[i] - '0');
    }
    if (id.size() > 2 && id[1] == '0') return -1;  // "%01" is not "%1"
    return v;
  }
  int find(const std::string& id) const {
    const int k = numeric(id);
    if (k >= 0) return static_cast<size_t>(k) < num.size() ? num[static_cast<size_t>(k)] : -1;
    auto it = other.find(id);
    return it == other.end() ? -1 : it->second;
  }
  void set(const std::string& id, int ref) {
    const int k = numeric(id);
    if (k >= 0) {
      if (static_cast<size_t>(k) >= num.size()) num.resize(static_cast<size_t>(k) + 1, -1);
      num[static_cast<size_t>(k)] = ref;
    } else {
      other[id] = ref;
    }
  }
};

Arg resolve_arg(const Value& x, State& st, const Env& env, int index) {
  Arg a;
  if (x.t == Value::Str && !x.s.empty() && x.s[0] == '%') {
    const int r = env.find(x.s);
    if (r < 0) throw ReplayErr{index, "unresolved reference " + x.s};
    a.ref = st.ref_at(r);
    return a;
  }
  if (x.t == Value::Arr) {
    a.is_list = true;
    for (const Value& i : x.a) a.list.push_back(resolve_arg(i, st, env, index));
    return a;
  }
  a.val = &x;
  return a;
}

void bind_outputs(const Value& instr, const std::vector<Ref*>& refs, Env& env, int index, const std::string& what) {
  const Value* outs = instr.get("outputs");
  static const Value empty = Value::arr();
  if (!outs) outs = &empty;
  if (outs->t != Value::Arr) defer("outputs");
  if (refs.size() != outs->a.size())
    throw ReplayErr{index, what + " produced " + std::to_string(refs.size()) + " outputs, trace recorded " +
                               std::to_string(outs->a.size())};
  for (size_t k = 0; k < refs.size(); ++k) {
    if (outs->a[k].t != Value::Str) defer("output id");
    env.set(outs->a[k].s, refs[k]->idx);
  }
}

// deserialize_trace (src/trace.py:95-125) of serialize_trace output
struct Parsed {
  std::vector<Value> instrs;
  bool have_hash = false;
  Value whash;
  std::string err;  // non-empty: not a trace the native replay takes (DEFER)
};
Parsed parse_trace(std::string_view text) {
  Parsed P;
  size_t pos = 0;
  int lineno = 0;
  while (pos < text.size()) {
    size_t nl = text.find('\n', pos);
    if (nl == std::string_view::npos) nl = text.size();
    std::string_view line = text.substr(pos, nl - pos);
    pos = nl + 1;
    ++lineno;
    bool blank = true;
    for (char c : line) blank &= (c == ' ' || c == '\t' || c == '\r');
    if (blank) continue;
    Value doc;
    if (!pj::parse(line, &doc) || doc.t != Value::Obj) {
      P.err = "unparsable trace line";
      return P;
    }
    if (doc.get("workload_hash") && !doc.get("op")) {
      if (lineno != 1) {
        P.err = "misplaced header";
        return P;
      }
      P.have_hash = true;
      P.whash = *doc.get("workload_hash");
      continue;
    }
    if (!doc.get("op")) {
      P.err = "missing op";
      return P;
    }
    P.instrs.push_back(std::move(doc));
  }
  return P;
}

void check_workload_hash(const Workload& w, const Parsed& P) {
  if (P.have_hash && P.whash.t != Value::Null) {
    bool same = P.whash.t == Value::Int &&
                (P.whash.big ? P.whash.s == std::to_string(w.hash)
                             : (P.whash.i >= 0 && static_cast<uint64_t>(P.whash.i) == w.hash));
    if (!same) throw ReplayErr{-1, "trace was recorded against a different workload (structural hash mismatch)"};
  }
}

// _step (src/trace.py:201-238) for one instruction
void step(State& st, Env& env, const Value& ins, int index) {
  const Value* opv = ins.get("op");
  if (opv->t != Value::Str) defer("op");
  const std::string& op = opv->s;
  static const Value empty_arr = Value::arr(), empty_obj = Value::obj();
  const Value* inputs = ins.get("inputs");
  if (!inputs) inputs = &empty_arr;
  if (inputs->t != Value::Arr) defer("inputs");
  const Value* attrs = ins.get("attrs");
  if (!attrs) attrs = &empty_obj;
  if (attrs->t != Value::Obj) defer("attrs");
  std::vector<Arg> args;
  args.reserve(inputs->a.size());
  for (const Value& x : inputs->a) args.push_back(resolve_arg(x, st, env, index));
  auto arg = [&](size_t i) -> const Arg& {
    if (i >= args.size()) defer("missing argument");
    return args[i];
  };
  const Value* decision = ins.get("decision");
#ifdef LSB_REPLAY_PROFILE
  auto prof_t0 = std::chrono::steady_clock::now();
  struct ProfEnd {
    const std::string& op;
    std::chrono::steady_clock::time_point t0;
    ~ProfEnd() { g_prof[op] += std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count(); }
  } prof_end{op, prof_t0};
#endif
  try {
    if (op == "get_blocks") {
      bind_outputs(ins, st.get_blocks(), env, index, op);
    } else if (op == "get_loops") {
      bind_outputs(ins, st.get_loops(arg(0)), env, index, op);
    } else if (op == "split") {
      bind_outputs(ins, st.split(arg(0), arg(1)), env, index, op);
    } else if (op == "fuse") {
      bind_outputs(ins, {st.fuse(arg(0))}, env, index, op);
    } else if (op == "reorder") {
      st.reorder(arg(0));
    } else if (op == "compute_at") {
      const Value* loc = attrs->get("location");
      if (loc && loc->t == Value::Str && loc->s == "root") st.compute_at(arg(0), nullptr);
      else st.compute_at(arg(0), &arg(1));
    } else if (op == "inline") {
      st.inline_block(arg(0));
    } else if (op == "parallelize") {
      st.parallelize(arg(0));
    } else if (op == "vectorize") {
      st.vectorize(arg(0));
    } else if (op == "unroll") {
      st.unroll(arg(0));
    } else if (op == "tensorize") {
      st.tensorize(arg(0), attrs->get("intrinsic"));
    } else if (op == "sample_perfect_tile") {
      if (!st.rng && (!decision || decision->t != Value::Obj)) defer("decision");
      bind_outputs(ins, st.sample_perfect_tile(arg(0), attrs->get("n"), st.rng ? nullptr : decision->get("tile")),
                   env, index, op);
    } else if (op == "sample_categorical") {
      if (!st.rng && (!decision || decision->t != Value::Obj)) defer("decision");
      bind_outputs(ins, {st.sample_categorical(attrs->get("candidates"), attrs->get("probs"),
                                               st.rng ? nullptr : decision->get("index"))},
                   env, index, op);
    } else if (op == "sample_compute_location") {
      if (!st.rng && (!decision || decision->t != Value::Obj)) defer("decision");
      bind_outputs(ins, {st.sample_compute_location(arg(0), st.rng ? nullptr : decision->get("index"))}, env, index,
                   op);
    } else {
      sched_err("unknown instruction op " + pj::py_repr(op));
    }
  } catch (const SchedErr& e) {
    throw ReplayErr{index, e.msg};
  }
}

Outcome finish(const State& st, const Parsed& P) {
  Outcome out;
  out.status = LS_REPLAY_ACCEPTED;
  out.program = serialize(st.prog);
  out.hash = structural_hash(st.prog);
  std::string& t = out.trace;
  if (P.have_hash) {
    Value h = Value::obj();
    h.put("workload_hash", P.whash);
    pj::dump(h, &t);
    t.push_back('\n');
  }
  t += st.text;
  return out;
}

Outcome rejected(const ReplayErr& e) {
  Outcome out;
  out.status = LS_REPLAY_REJECTED;
  out.index = e.index;
  out.reason = e.reason;
  return out;
}

Outcome replay_one(const Workload& w, std::string_view text, const uint64_t* resample_seed = nullptr) {
  Parsed P = parse_trace(text);
  Outcome out;
  if (!P.err.empty()) {
    out.reason = P.err;
    return out;
  }
  try {
    check_workload_hash(w, P);
    State st(local_e0(w), &w.loop_vars);
    if (resample_seed) st.rng = std::make_shared<PyRandom>(*resample_seed);
    Env env;
    for (int index = 0; index < static_cast<int>(P.instrs.size()); ++index)
      step(st, env, P.instrs[static_cast<size_t>(index)], index);
    return finish(st, P);
  } catch (const ReplayErr& e) {
    return rejected(e);
  } catch (const Defer& d) {
    out.status = LS_REPLAY_DEFER;
    out.reason = d.msg;
  }
  return out;
}

// ---------------------------------------------------------------------------
// single-decision neighbourhoods (the look-ahead of SURVEY.md §8f-2): every
// trace `mutate` (src/trace.py:287-309) can propose from a member, as the
// reference would serialize it, so a prefetched result is found under the
// exact key _Validator.candidate computes
// ---------------------------------------------------------------------------

struct Fp {
  uint64_t a, b;
  bool operator==(const Fp& o) const { return a == o.a && b == o.b; }
};
struct FpHash {
  size_t operator()(const Fp& f) const { return static_cast<size_t>(f.a ^ (f.b * 0x9E3779B97F4A7C15ULL)); }
};
Fp fingerprint(std::string_view s) {
  uint64_t a = 1469598103934665603ULL, b = 0x84222325cbf29ce4ULL;
  for (unsigned char c : s) {
    a = (a ^ c) * 1099511628211ULL;
    b = (b ^ c) * 0x100000001b3ULL + 0x9E3779B97F4A7C15ULL;
    b ^= b >> 29;
  }
  return {a, b};
}

// ordered n-tuples of positive integers with product `extent`
// (ordered_factorizations, src/schedule.py:77-88; order irrelevant here)
void factorizations(int64_t extent, int64_t n, std::vector<int64_t>& cur, std::vector<std::vector<int64_t>>* out) {
  if (n == 1) {
    cur.push_back(extent);
    out->push_back(cur);
    cur.pop_back();
    return;
  }
  for (int64_t d = 1; d <= extent; ++d)
    if (extent % d == 0) {
      cur.push_back(d);
      factorizations(extent / d, n - 1, cur, out);
      cur.pop_back();
    }
}

// the alternative decisions of one sampling instruction (_mutation_domain,
// src/trace.py:268-284) as rewritten instruction lines; false when the line
// is not a sampling instruction the enumeration understands
struct Alt {
  Value ins;         // the instruction with the alternative decision
  std::string line;  // its serialize_trace line
};
bool neighbour_lines(const Value& ins, std::vector<Alt>* out) {
  const Value* op = ins.get("op");
  const Value* dec = ins.get("decision");
  const Value* attrs = ins.get("attrs");
  if (!op || op->t != Value::Str || !dec || dec->t != Value::Obj || !attrs || attrs->t != Value::Obj) return false;
  auto with = [&](const char* key, Value v, const char* key2 = nullptr, Value v2 = Value()) {
    Value x = ins;
    Value* d = nullptr;
    for (auto& kv : x.o)
      if (kv.first == "decision") d = &kv.second;
    bool set1 = false, set2 = false;
    for (auto& kv : d->o) {
      if (kv.first == key) { kv.second = v; set1 = true; }
      if (key2 && kv.first == key2) { kv.second = v2; set2 = true; }
    }
    if (!set1) d->put(key, v);
    if (key2 && !set2) d->put(key2, v2);
    std::string line = pj::dumps(x);
    out->push_back({std::move(x), std::move(line)});
  };
  if (op->s == "sample_perfect_tile") {
    const Value* e = attrs->get("extent");
    const Value* n = attrs->get("n");
    const Value* tile = dec->get("tile");
    if (!e || !n || !tile || e->t != Value::Int || n->t != Value::Int || tile->t != Value::Arr || e->big || n->big ||
        e->i < 1 || n->i < 1 || n->i > 8)
      return false;
    std::vector<int64_t> cur_tile;
    for (const Value& x : tile->a) {
      if (x.t != Value::Int || x.big) return false;
      cur_tile.push_back(x.i);
    }
    std::vector<std::vector<int64_t>> dom;
    std::vector<int64_t> cur;
    factorizations(e->i, n->i, cur, &dom);
    for (const auto& f : dom) {
      if (f == cur_tile) continue;
      Value l = Value::arr();
      for (int64_t x : f) l.a.push_back(Value::integer(x));
      with("tile", std::move(l));
    }
    return true;
  }
  if (op->s == "sample_categorical") {
    const Value* probs = attrs->get("probs");
    const Value* idx = dec->get("index");
    if (!probs || probs->t != Value::Arr || !idx || idx->t != Value::Int) return false;
    std::vector<double> w;
    for (const Value& p : probs->a) {
      if (p.t == Value::Float) w.push_back(p.d);
      else if (p.t == Value::Int && !p.big) w.push_back(static_cast<double>(p.i));
      else return false;
    }
    double total = 0;
    for (double x : w) total += x;
    for (size_t i = 0; i < w.size(); ++i) {
      if (!(w[i] > 0) || static_cast<int64_t>(i) == idx->i) continue;
      with("index", Value::integer(static_cast<int64_t>(i)), "prob", Value::real(w[i] / total));
    }
    return true;
  }
  if (op->s == "sample_compute_location") {
    const Value* size = dec->get("size");
    const Value* idx = dec->get("index");
    if (!size || !idx || size->t != Value::Int || idx->t != Value::Int || size->big) return false;
    for (int64_t i = 0; i < size->i; ++i)
      if (i != idx->i) with("index", Value::integer(i));
    return true;
  }
  return false;
}

char* dup_cstr(const std::string& s) {
  char* p = static_cast<char*>(std::malloc(s.size() + 1));
  if (p) std::memcpy(p, s.c_str(), s.size() + 1);
  return p;
}

}  // namespace rp
}  // namespace lsb

using namespace lsb;

struct ls_replayer {
  rp::Workload w;
  // keys of every trace replayed through ls_replay_neighbours (128-bit
  // fingerprints): a later expansion replays only new neighbours
  std::mutex seen_mu;
  std::unordered_set<rp::Fp, rp::FpHash> seen;
  std::unordered_set<uint64_t> hashes;  // structural hashes already handed out
};

struct ls_neighbours {
  struct Item {
    uint64_t hash;
    std::string program;
  };
  std::vector<Item> items;  // programs of structural hashes not seen before
  int64_t replayed = 0, accepted = 0, rejected = 0, deferred = 0;
};

extern "C" {

ls_status ls_replayer_create(const char* e0, size_t len, ls_replayer** out) {
  if (!e0 || !out) {
    set_error("ls_replayer_create: null argument");
    return LS_ERR_ARG;
  }
  auto r = std::make_unique<ls_replayer>();
  if (!rp::program_from(std::string_view(e0, len), &r->w.e0)) {
    set_error("ls_replayer_create: workload text is not a serialized program");
    return LS_ERR_PARSE;
  }
  if (!rp::validate_ir(r->w.e0).empty()) {
    set_error("ls_replayer_create: workload program is not valid IR");
    return LS_ERR_PARSE;
  }
  r->w.hash = rp::structural_hash(r->w.e0);
  r->w.text.assign(e0, len);
  static std::atomic<uint64_t> serials{1};
  r->w.serial = serials.fetch_add(1);
  rp::iter_stmts(r->w.e0.root, [&](const rp::Path&, const rp::St& s) {
    if (s.k == rp::S_LOOP) r->w.loop_vars.insert(s.var);
  });
  *out = r.release();
  return LS_OK;
}

ls_status ls_replayer_hash(ls_replayer* r, uint64_t* out) {
  if (!r || !out) {
    set_error("ls_replayer_hash: null argument");
    return LS_ERR_ARG;
  }
  *out = r->w.hash;
  return LS_OK;
}

ls_status ls_replay_batch(ls_replayer* r, const char* const* traces, const size_t* lens, int n,
                          ls_replay_result* out) {
  if (!r || n < 0 || (n > 0 && (!traces || !lens || !out))) {
    set_error("ls_replay_batch: bad arguments");
    return LS_ERR_ARG;
  }
  auto one = [&](int i) {
    rp::Outcome o = rp::replay_one(r->w, std::string_view(traces[i], lens[i]));
    ls_replay_result& x = out[i];
    x.status = o.status;
    x.index = o.index;
    x.hash = o.hash;
    x.program = o.status == LS_REPLAY_ACCEPTED ? rp::dup_cstr(o.program) : nullptr;
    x.trace = o.status == LS_REPLAY_ACCEPTED ? rp::dup_cstr(o.trace) : nullptr;
    x.reason = o.status != LS_REPLAY_ACCEPTED ? rp::dup_cstr(o.reason) : nullptr;
  };
  if (n >= 8) HostPool::get().run(n, one);
  else
    for (int i = 0; i < n; ++i) one(i);
  return LS_OK;
}

void ls_replay_free(ls_replay_result* res, int n) {
  if (!res) return;
  for (int i = 0; i < n; ++i) {
    std::free(res[i].program);
    std::free(res[i].trace);
    std::free(res[i].reason);
    res[i].program = res[i].trace = res[i].reason = nullptr;
  }
}

ls_status ls_replay_resample(ls_replayer* r, const char* trace, size_t len, uint64_t seed, ls_replay_result* out) {
  if (!r || !trace || !out) {
    set_error("ls_replay_resample: bad arguments");
    return LS_ERR_ARG;
  }
  rp::Outcome o = rp::replay_one(r->w, std::string_view(trace, len), &seed);
  out->status = o.status;
  out->index = o.index;
  out->hash = o.hash;
  out->program = o.status == LS_REPLAY_ACCEPTED ? rp::dup_cstr(o.program) : nullptr;
  out->trace = o.status == LS_REPLAY_ACCEPTED ? rp::dup_cstr(o.trace) : nullptr;
  out->reason = o.status != LS_REPLAY_ACCEPTED ? rp::dup_cstr(o.reason) : nullptr;
  return LS_OK;
}

ls_status ls_program_hash(const char* program, size_t len, uint64_t* out) {
  rp::Prog p;
  if (!program || !out || !rp::program_from(std::string_view(program, len), &p)) {
    set_error("ls_program_hash: not a serialized program");
    return LS_ERR_PARSE;
  }
  *out = rp::structural_hash(p);
  return LS_OK;
}

void ls_replayer_destroy(ls_replayer* r) { delete r; }

ls_status ls_replay_neighbours(ls_replayer* r, const char* const* traces, const size_t* lens, int n,
                               ls_neighbours** out) {
  if (!r || !out || n < 0 || (n > 0 && (!traces || !lens))) {
    set_error("ls_replay_neighbours: bad arguments");
    return LS_ERR_ARG;
  }
  // per member: the new neighbours (deduplicated against every key this
  // replayer has expanded), then one replay of the member that snapshots the
  // state before each mutated instruction, so a neighbour replays only the
  // suffix from its changed decision
  struct Res {
    std::vector<rp::Outcome> outs;
  };
  std::vector<Res> per(static_cast<size_t>(n));
  auto one = [&](int m) {
    std::string_view text(traces[m], lens[m]);
    rp::Parsed P = rp::parse_trace(text);
    if (!P.err.empty()) return;
    std::vector<std::string_view> lines;
    size_t pos = 0;
    while (pos < text.size()) {
      size_t nl = text.find('\n', pos);
      if (nl == std::string_view::npos) nl = text.size();
      lines.push_back(text.substr(pos, nl - pos));
      pos = nl + 1;
    }
    const size_t hdr = P.have_hash ? 1 : 0;
    if (lines.size() != P.instrs.size() + hdr) return;  // blank lines: leave to the sequential path
    struct Job {
      int at;
      rp::Value ins;
      std::string key;
    };
    std::vector<Job> jobs;
    for (size_t j = 0; j < P.instrs.size(); ++j) {
      std::vector<rp::Alt> alts;
      if (!rp::neighbour_lines(P.instrs[j], &alts)) continue;
      for (auto& alt : alts) {
        std::string key;
        key.reserve(text.size() + 64);
        for (size_t k = 0; k < lines.size(); ++k) {
          if (k == j + hdr) key += alt.line;
          else key.append(lines[k].data(), lines[k].size());
          key.push_back('\n');
        }
        jobs.push_back({static_cast<int>(j), std::move(alt.ins), std::move(key)});
      }
    }
    {
      std::lock_guard<std::mutex> lk(r->seen_mu);
      r->seen.insert(rp::fingerprint(text));
      std::vector<Job> fresh;
      for (auto& jb : jobs)
        if (r->seen.insert(rp::fingerprint(jb.key)).second) fresh.push_back(std::move(jb));
      jobs.swap(fresh);
    }
    if (jobs.empty()) return;
    auto& items = per[static_cast<size_t>(m)].outs;
    try {
      rp::check_workload_hash(r->w, P);
    } catch (const rp::ReplayErr& e) {
      for (size_t k = 0; k < jobs.size(); ++k) items.push_back(rp::rejected(e));
      return;
    }
    // the member, with snapshots before every mutated position
    std::map<int, std::pair<rp::State, rp::Env>> snap;
    for (const auto& jb : jobs) snap.emplace(jb.at, std::make_pair(rp::State(rp::local_e0(r->w), &r->w.loop_vars), rp::Env()));
    rp::State st(rp::local_e0(r->w), &r->w.loop_vars);
    rp::Env env;
    int failed_at = static_cast<int>(P.instrs.size());
    rp::Outcome member_fail;
    try {
      for (int index = 0; index < static_cast<int>(P.instrs.size()); ++index) {
        auto it = snap.find(index);
        if (it != snap.end()) it->second = std::make_pair(st, env);
        rp::step(st, env, P.instrs[static_cast<size_t>(index)], index);
      }
    } catch (const rp::ReplayErr& e) {
      failed_at = e.index;
      member_fail = rp::rejected(e);
    } catch (const rp::Defer& d) {
      failed_at = -1;  // leave every neighbour to the sequential path
    }
    for (auto& jb : jobs) {
      if (failed_at < 0) break;
      if (jb.at > failed_at) {  // same prefix up to the member's failure: the same verdict
        items.push_back(member_fail);
        continue;
      }
      rp::Outcome o;
      try {
        auto& sn = snap.at(jb.at);
        rp::State s2 = sn.first;
        rp::Env e2 = sn.second;
        rp::step(s2, e2, jb.ins, jb.at);
        for (int index = jb.at + 1; index < static_cast<int>(P.instrs.size()); ++index)
          rp::step(s2, e2, P.instrs[static_cast<size_t>(index)], index);
        o = rp::finish(s2, P);
      } catch (const rp::ReplayErr& e) {
        o = rp::rejected(e);
      } catch (const rp::Defer& d) {
        o.status = LS_REPLAY_DEFER;
        o.reason = d.msg;
      }
      items.push_back(std::move(o));
    }
  };
  if (n > 1) HostPool::get().run(n, one);
  else if (n == 1) one(0);
  auto nb = std::make_unique<ls_neighbours>();
  std::lock_guard<std::mutex> lk(r->seen_mu);
  for (auto& v : per)
    for (auto& o : v.outs) {
      ++nb->replayed;
      if (o.status == LS_REPLAY_ACCEPTED) {
        ++nb->accepted;
        if (r->hashes.insert(o.hash).second) nb->items.push_back({o.hash, std::move(o.program)});
      } else if (o.status == LS_REPLAY_REJECTED) {
        ++nb->rejected;
      } else {
        ++nb->deferred;
      }
    }
  *out = nb.release();
  return LS_OK;
}

ls_status ls_neighbours_count(ls_neighbours* nb, int* count) {
  if (!nb || !count) {
    set_error("ls_neighbours_count: null argument");
    return LS_ERR_ARG;
  }
  *count = static_cast<int>(nb->items.size());
  return LS_OK;
}

ls_status ls_neighbours_get(ls_neighbours* nb, int i, uint64_t* hash, const char** program) {
  if (!nb || i < 0 || static_cast<size_t>(i) >= nb->items.size() || !hash || !program) {
    set_error("ls_neighbours_get: bad arguments");
    return LS_ERR_ARG;
  }
  *hash = nb->items[static_cast<size_t>(i)].hash;
  *program = nb->items[static_cast<size_t>(i)].program.c_str();
  return LS_OK;
}

ls_status ls_neighbours_stats(ls_neighbours* nb, int64_t* out4) {
  if (!nb || !out4) {
    set_error("ls_neighbours_stats: null argument");
    return LS_ERR_ARG;
  }
  out4[0] = nb->replayed;
  out4[1] = nb->accepted;
  out4[2] = nb->rejected;
  out4[3] = nb->deferred;
  return LS_OK;
}

void ls_neighbours_destroy(ls_neighbours* nb) { delete nb; }

}  // extern "C"
