// JSON front end + IR analysis helpers.  See ir.hpp.
#include "ir.hpp"

#include <cctype>
#include <cstdlib>
#include <cstring>

namespace lsb {

namespace {

const IntrinsicInfo kIntrinsics[] = {{"tu.mma4", 4, 128, 48}};

// ---- a small JSON reader specialised to the program schema ---------------
// Values are read straight into IR nodes; objects are scanned key by key so
// key order (the reference writes sort_keys=True) does not matter.
class Reader {
 public:
  Reader(std::string_view s, Program* p) : s_(s), p_(p) {}
  bool good() const { return err_.empty(); }
  const std::string& error() const { return err_; }

  bool parse_top() {
    ws();
    if (!expect('{')) return false;
    bool have_buffers = false, have_root = false;
    std::string root_text_key;
    // Two passes would be simpler but programs reference buffers by name in
    // loads, so buffers must be known first: remember the root's span.
    size_t root_begin = 0, root_end = 0;
    for (bool first = true;; first = false) {
      ws();
      if (peek() == '}') { ++i_; break; }
      if (!first && !expect(',')) return false;
      std::string key;
      if (!string(&key) || !expect(':')) return false;
      if (key == "buffers") {
        have_buffers = true;
        if (!buffers()) return false;
      } else if (key == "root") {
        have_root = true;
        ws();
        root_begin = i_;
        if (!skip_value()) return false;
        root_end = i_;
      } else if (!skip_value()) {
        return false;
      }
    }
    if (!have_buffers || !have_root) return fail("missing 'buffers' or 'root'");
    size_t save = i_;
    i_ = root_begin;
    bool r = stmt_list(&p_->root);
    if (r && i_ != root_end) return fail("trailing data in root");
    i_ = save;
    return r;
  }

 private:
  std::string_view s_;
  Program* p_;
  size_t i_ = 0;
  std::string err_;

  bool fail(const char* m) {
    if (err_.empty()) err_ = std::string(m) + " at offset " + std::to_string(i_);
    return false;
  }
  void ws() { while (i_ < s_.size() && (s_[i_] == ' ' || s_[i_] == '\n' || s_[i_] == '\t' || s_[i_] == '\r')) ++i_; }
  char peek() { ws(); return i_ < s_.size() ? s_[i_] : '\0'; }
  bool expect(char c) {
    ws();
    if (i_ >= s_.size() || s_[i_] != c) return fail("unexpected character");
    ++i_;
    return true;
  }
  bool string(std::string* out) {
    ws();
    if (i_ >= s_.size() || s_[i_] != '"') return fail("expected string");
    ++i_;
    out->clear();
    while (i_ < s_.size() && s_[i_] != '"') {
      if (s_[i_] == '\\') { ++i_; if (i_ >= s_.size()) break; }
      out->push_back(s_[i_++]);
    }
    if (i_ >= s_.size()) return fail("unterminated string");
    ++i_;
    return true;
  }
  bool integer(int64_t* v) {
    ws();
    size_t j = i_;
    const bool neg = j < s_.size() && s_[j] == '-';
    if (neg) ++j;
    const size_t d0 = j;
    uint64_t x = 0;
    while (j < s_.size() && s_[j] >= '0' && s_[j] <= '9' && j - d0 < 19) x = x * 10 + static_cast<uint64_t>(s_[j++] - '0');
    if (j == d0) return fail("expected integer");
    if (j < s_.size() && (s_[j] == '.' || s_[j] == 'e' || s_[j] == 'E' || (s_[j] >= '0' && s_[j] <= '9')))
      return fail("non-integer number");  // fractions, exponents, more than 18 digits
    i_ = j;
    *v = neg ? -static_cast<int64_t>(x) : static_cast<int64_t>(x);
    return true;
  }
  // a string skipped in place (no copy): the first pass over the root and
  // unknown keys only need its end
  bool skip_string() {
    ws();
    if (i_ >= s_.size() || s_[i_] != '"') return fail("expected string");
    ++i_;
    while (i_ < s_.size() && s_[i_] != '"') i_ += s_[i_] == '\\' ? 2 : 1;
    if (i_ >= s_.size()) return fail("unterminated string");
    ++i_;
    return true;
  }
  bool skip_value() {
    char c = peek();
    if (c == '"') return skip_string();
    if (c == '{' || c == '[') {
      char close = c == '{' ? '}' : ']';
      ++i_;
      for (bool first = true;; first = false) {
        if (peek() == close) { ++i_; return true; }
        if (!first && !expect(',')) return false;
        if (c == '{' && (!skip_string() || !expect(':'))) return false;
        if (!skip_value()) return false;
      }
    }
    if (c == '-' || (c >= '0' && c <= '9')) {
      ++i_;
      while (i_ < s_.size() && (std::isdigit(static_cast<unsigned char>(s_[i_])) || s_[i_] == '.' ||
                                 s_[i_] == 'e' || s_[i_] == 'E' || s_[i_] == '-' || s_[i_] == '+'))
        ++i_;
      return true;
    }
    for (const char* lit : {"null", "true", "false"}) {
      size_t n = std::strlen(lit);
      if (s_.substr(i_, n) == lit) { i_ += n; return true; }
    }
    return fail("bad value");
  }
  template <class F>
  bool array(F&& each) {
    if (!expect('[')) return false;
    for (bool first = true;; first = false) {
      if (peek() == ']') { ++i_; return true; }
      if (!first && !expect(',')) return false;
      if (!each()) return false;
    }
  }
  // object keys of the interchange format never contain escapes: view them
  // in place instead of copying each into a std::string
  bool key(std::string_view* out) {
    ws();
    if (i_ >= s_.size() || s_[i_] != '"') return fail("expected string");
    const size_t b = ++i_;
    while (i_ < s_.size() && s_[i_] != '"') {
      if (s_[i_] == '\\') return fail("escaped object key");
      ++i_;
    }
    if (i_ >= s_.size()) return fail("unterminated string");
    *out = s_.substr(b, i_ - b);
    ++i_;
    return true;
  }
  template <class F>
  bool object(F&& each_key) {
    if (!expect('{')) return false;
    for (bool first = true;; first = false) {
      if (peek() == '}') { ++i_; return true; }
      if (!first && !expect(',')) return false;
      std::string_view k;
      if (!key(&k) || !expect(':')) return false;
      if (!each_key(k)) return false;
    }
  }

  bool buffers() {
    return array([&] {
      Buffer b;
      bool ok = object([&](std::string_view k) {
        if (k == "name") return string(&b.name);
        if (k == "role") {
          std::string r;
          if (!string(&r)) return false;
          b.role = r == "input" ? 0 : r == "output" ? 1 : 2;
          return true;
        }
        if (k == "shape")
          return array([&] { int64_t v; if (!integer(&v)) return false; b.shape.push_back(v); return true; });
        return skip_value();
      });
      p_->buffers.push_back(std::move(b));
      return ok;
    });
  }

  // names (loop variables, buffers) carry no escapes in the interchange
  // format, so they are read as views (key()) and only copied when new
  int var_id(std::string_view name) {
    for (size_t i = 0; i < p_->vars.size(); ++i)
      if (p_->vars[i] == name) return static_cast<int>(i);
    p_->vars.emplace_back(name);
    return static_cast<int>(p_->vars.size()) - 1;
  }
  int buf_id(std::string_view name) {
    int b = p_->buffer_id(name);
    if (b < 0) fail("unknown buffer");
    return b;
  }

  bool expr_list(std::vector<Expr*>* out) {
    out->reserve(4);  // operands / index lists are short: one allocation instead of up to three
    return array([&] { Expr* e = expr(); if (!e) return false; out->push_back(e); return true; });
  }

  Expr* expr() {
    Expr* e = p_->new_expr();
    bool ok = object([&](std::string_view k) {
      if (k == "int") { e->op = Op::Int; return integer(&e->value); }
      if (k == "var") { std::string_view n; if (!key(&n)) return false; e->op = Op::Var; e->var = var_id(n); return true; }
      if (k == "load") {
        e->op = Op::Load;
        return object([&](std::string_view lk) {
          if (lk == "buffer") { std::string_view n; if (!key(&n)) return false; e->buffer = buf_id(n); return good(); }
          if (lk == "indices") return expr_list(&e->kids);
          return skip_value();
        });
      }
      static const char* kBin[] = {"add", "sub", "mul", "max", "min", "floordiv", "mod"};
      for (int b = 0; b < 7; ++b)
        if (k == kBin[b]) { e->op = static_cast<Op>(static_cast<int>(Op::Add) + b); return expr_list(&e->kids); }
      if (k == "select") { e->op = Op::Select; return expr_list(&e->kids); }
      return fail("unknown expression tag");
    });
    if (!ok) return nullptr;
    size_t want = e->op == Op::Select ? 3 : (e->op >= Op::Add ? 2 : e->kids.size());
    if (e->kids.size() != want) { fail("wrong operand count"); return nullptr; }
    return e;
  }

  bool stmt_list(std::vector<Stmt*>* out) {
    return array([&] { Stmt* s = stmt(); if (!s) return false; out->push_back(s); return true; });
  }

  Stmt* stmt() {
    Stmt* s = p_->new_stmt();
    bool ok = object([&](std::string_view k) {
      if (k == "loop") {
        s->type = SType::Loop;
        return object([&](std::string_view lk) {
          if (lk == "var") { std::string_view n; if (!key(&n)) return false; s->var = var_id(n); return true; }
          if (lk == "extent") return integer(&s->extent);
          if (lk == "kind") {
            std::string kd;
            if (!string(&kd)) return false;
            if (kd == "serial") s->kind = Kind::Serial;
            else if (kd == "parallel") s->kind = Kind::Parallel;
            else if (kd == "vectorized") s->kind = Kind::Vectorized;
            else if (kd == "unrolled") s->kind = Kind::Unrolled;
            else return fail("unknown loop kind");
            return true;
          }
          if (lk == "body") return stmt_list(&s->body);
          return skip_value();
        });
      }
      if (k == "compute") {
        s->type = SType::Compute;
        return object([&](std::string_view ck) {
          if (ck == "name") return string(&s->name);
          if (ck == "buffer") { std::string_view n; if (!key(&n)) return false; s->buffer = buf_id(n); return good(); }
          if (ck == "indices") return expr_list(&s->indices);
          if (ck == "value") return (s->value = expr()) != nullptr;
          if (ck == "init") return (s->init = expr()) != nullptr;
          if (ck == "epilogue") return (s->epilogue = expr()) != nullptr;
          return skip_value();
        });
      }
      if (k == "intrinsic") {
        s->type = SType::Intrinsic;
        return object([&](std::string_view ik) {
          if (ik == "name") {
            std::string n;
            if (!string(&n)) return false;
            int cnt = 0;
            const IntrinsicInfo* reg = intrinsic_registry(&cnt);
            for (int r = 0; r < cnt; ++r)
              if (n == reg[r].name) s->intrinsic = r;
            if (s->intrinsic < 0) return fail("unknown intrinsic");
            return true;
          }
          if (ik == "block") return string(&s->name);
          if (ik == "init") return (s->init = expr()) != nullptr;
          if (ik == "operands")
            return array([&] {
              int buf = -1;
              std::vector<Expr*> idx;
              bool r = object([&](std::string_view ok2) {
                if (ok2 == "buffer") { std::string_view n; if (!key(&n)) return false; buf = buf_id(n); return good(); }
                if (ok2 == "indices") return expr_list(&idx);
                return skip_value();
              });
              s->op_buffers.push_back(buf);
              s->op_indices.push_back(std::move(idx));
              return r;
            });
          return skip_value();
        });
      }
      return fail("unknown statement tag");
    });
    if (!ok) return nullptr;
    if (s->type == SType::Compute && (!s->value || s->buffer < 0)) { fail("incomplete compute"); return nullptr; }
    return s;
  }
};

void walk_blocks(Stmt* s, std::vector<Stmt*>* loops, std::vector<Block>* out) {
  if (s->type == SType::Loop) {
    loops->push_back(s);
    for (Stmt* c : s->body) walk_blocks(c, loops, out);
    loops->pop_back();
    return;
  }
  out->push_back(Block{s, *loops});
}

}  // namespace

const IntrinsicInfo* intrinsic_registry(int* n) {
  *n = static_cast<int>(sizeof(kIntrinsics) / sizeof(kIntrinsics[0]));
  return kIntrinsics;
}

int Program::buffer_id(std::string_view name) const {
  for (size_t i = 0; i < buffers.size(); ++i)
    if (buffers[i].name == name) return static_cast<int>(i);
  return -1;
}

std::unique_ptr<Program> parse_program(std::string_view text, std::string* err) {
  auto p = std::make_unique<Program>();
  Reader r(text, p.get());
  if (!r.parse_top() || !r.good()) {
    if (err) *err = r.error().empty() ? "parse error" : r.error();
    return nullptr;
  }
  return p;
}

std::vector<Block> blocks_preorder(const Program& p) {
  std::vector<Block> out;
  std::vector<Stmt*> loops;
  for (Stmt* s : p.root) walk_blocks(s, &loops, &out);
  return out;
}

void expr_vars(const Expr* e, std::vector<int>* out) {
  if (!e) return;
  if (e->op == Op::Var) { out->push_back(e->var); return; }
  for (const Expr* k : e->kids) expr_vars(k, out);
}

int64_t arith_ops(const Expr* e) {
  if (!e) return 0;
  switch (e->op) {
    case Op::Int: case Op::Var: case Op::Load: return 0;
    default: {
      int64_t n = 1;
      for (const Expr* k : e->kids) n += arith_ops(k);
      return n;
    }
  }
}

void collect_loads(const Expr* e, std::vector<const Expr*>* out) {
  if (!e) return;
  if (e->op == Op::Load) out->push_back(e);
  for (const Expr* k : e->kids) collect_loads(k, out);
}

bool affine_coeffs(const Expr* e, size_t nvars, std::vector<int64_t>* coeff, int64_t* c0) {
  coeff->assign(nvars, 0);
  *c0 = 0;
  switch (e->op) {
    case Op::Int: *c0 = e->value; return true;
    case Op::Var: (*coeff)[e->var] = 1; return true;
    case Op::Add: case Op::Sub: case Op::Mul: break;
    default: return false;
  }
  std::vector<int64_t> ca, cb;
  int64_t a0, b0;
  if (!affine_coeffs(e->kids[0], nvars, &ca, &a0) || !affine_coeffs(e->kids[1], nvars, &cb, &b0)) return false;
  if (e->op != Op::Mul) {
    int64_t sg = e->op == Op::Add ? 1 : -1;
    for (size_t v = 0; v < nvars; ++v) (*coeff)[v] = ca[v] + sg * cb[v];
    *c0 = a0 + sg * b0;
    return true;
  }
  bool av = false, bv = false;
  for (size_t v = 0; v < nvars; ++v) { av |= ca[v] != 0; bv |= cb[v] != 0; }
  if (av && bv) return false;
  const std::vector<int64_t>& vv = bv ? cb : ca;
  int64_t scale = bv ? a0 : b0;
  for (size_t v = 0; v < nvars; ++v) (*coeff)[v] = vv[v] * scale;
  *c0 = a0 * b0;
  return true;
}

}  // namespace lsb
