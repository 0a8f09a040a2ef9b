// Planner for general workloads.  See affine.hpp.
#include "affine.hpp"

#include <algorithm>
#include <cstring>
#include <random>

#include "plan.hpp"

namespace lsb {

namespace {

const int64_t kATiles[] = {1, 2, 3, 4, 6, 7, 8, 12, 14, 16};
constexpr int kNATiles = 10;

// witness kinds: the access whose index at `dim` is exactly the axis variable
enum WKind { W_STORE = 0, W_Y = 1, W_X = 2 };

bool fail(std::string* err, const std::string& m) {
  if (err) *err = m;
  return false;
}

int exact_dim(const std::vector<Expr*>& idx, int var) {
  for (size_t d = 0; d < idx.size(); ++d)
    if (idx[d]->op == Op::Var && idx[d]->var == var) return static_cast<int>(d);
  return -1;
}

bool has_var(const std::vector<Expr*>& idx, int var) {
  std::vector<int> vs;
  for (const Expr* e : idx) expr_vars(e, &vs);
  return std::find(vs.begin(), vs.end(), var) != vs.end();
}

int64_t host_eval(const Expr* e, const std::vector<int64_t>& vals, bool* ok) {
  switch (e->op) {
    case Op::Int: return e->value;
    case Op::Var: return vals[static_cast<size_t>(e->var)];
    case Op::Load: *ok = false; return 0;
    case Op::Select: {
      int64_t c = host_eval(e->kids[0], vals, ok);
      return c != 0 ? host_eval(e->kids[1], vals, ok) : host_eval(e->kids[2], vals, ok);
    }
    default: break;
  }
  int64_t a = host_eval(e->kids[0], vals, ok), b = host_eval(e->kids[1], vals, ok);
  switch (e->op) {
    case Op::Add: return a + b;
    case Op::Sub: return a - b;
    case Op::Mul: return a * b;
    case Op::Max: return std::max(a, b);
    case Op::Min: return std::min(a, b);
    case Op::FloorDiv: { int64_t q = a / b; if ((a % b) && ((a < 0) != (b < 0))) --q; return q; }
    case Op::Mod: { int64_t r = a % b; if (r && ((r < 0) != (b < 0))) r += b; return r; }
    default: *ok = false; return 0;
  }
}

// The X-side factor of a contraction value: a Load, or Select(cond, Load, 0).
bool x_side(const Expr* f, const Expr** load, const Expr** cond) {
  if (f->op == Op::Load) { *load = f; *cond = nullptr; return true; }
  if (f->op == Op::Select && f->kids[1]->op == Op::Load && f->kids[2]->op == Op::Int && f->kids[2]->value == 0) {
    *load = f->kids[1];
    *cond = f->kids[0];
    return true;
  }
  return false;
}

GeneralPlan unsupported(const char* why) {
  GeneralPlan g;
  g.status = P_UNSUPPORTED;
  g.why = why;
  return g;
}

}  // namespace

int simta_tile_index(int64_t v) {
  for (int i = 0; i < kNATiles; ++i)
    if (kATiles[i] == v) return i;
  return -1;
}

bool simta_tile_supported(int64_t rm, int64_t rn) {
  return simta_tile_index(rm) >= 0 && simta_tile_index(rn) >= 0 && rm * rn <= 64;
}

bool analyze_general(const Program& e0, GeneralWorkload* w, std::string* err) {
  std::vector<Block> blocks = blocks_preorder(e0);
  const Block* con = nullptr;
  for (const Block& b : blocks) {
    if (b.stmt->type != SType::Compute) return fail(err, "intrinsic blocks are not supported");
    if (b.stmt->init) {
      if (con) return fail(err, "more than one reduction block");
      con = &b;
    }
  }
  if (!con) return fail(err, "no contraction block");
  const Stmt* s = con->stmt;
  if (s->init->op != Op::Int || s->init->value != 0 || s->epilogue)
    return fail(err, "contraction must start from 0 without an epilogue in e0");
  const Expr* v = s->value;
  if (v->op != Op::Mul || v->kids[0]->op != Op::Load || v->kids[1]->op != Op::Load)
    return fail(err, "contraction value must be a product of two loads");
  const Expr* a = v->kids[0];
  const Expr* b = v->kids[1];
  w->block = s->name;
  w->x_buf = e0.buffers[static_cast<size_t>(a->buffer)].name;
  w->y_buf = e0.buffers[static_cast<size_t>(b->buffer)].name;
  w->c_buf = e0.buffers[static_cast<size_t>(s->buffer)].name;
  for (const Stmt* l : con->loops) {
    bool sp = has_var(s->indices, l->var);
    bool in_a = has_var(a->kids, l->var), in_b = has_var(b->kids, l->var);
    int group;
    if (sp) group = in_a && in_b ? AG_B : in_a ? AG_M : in_b ? AG_N : -1;
    else group = (in_a || in_b) ? AG_K : -1;
    if (group < 0) return fail(err, "loop variable outside the contraction pattern");
    std::string wb;
    int wd = -1;
    if (sp && (wd = exact_dim(s->indices, l->var)) >= 0) wb = "store";
    else if ((wd = exact_dim(b->kids, l->var)) >= 0) wb = "y";
    else if ((wd = exact_dim(a->kids, l->var)) >= 0) wb = "x";
    else return fail(err, "no access indexed by exactly one axis variable");
    w->axis_var.push_back(e0.vars[static_cast<size_t>(l->var)]);
    w->axis_group.push_back(group);
    w->axis_extent.push_back(l->extent);
    w->wit_buf.push_back(wb);
    w->wit_dim.push_back(wd);
  }
  for (const Buffer& B : e0.buffers) {
    w->buffers.push_back(B.name);
    w->shapes.push_back(B.shape);
    w->roles.push_back(B.role);
    if (B.name == w->c_buf) {
      int64_t n = 1;
      for (int64_t x : B.shape) n *= x;
      w->c_elems = n;
    }
  }
  return true;
}

namespace {

struct LoopPart { int axis; int64_t ext, stride; Kind kind; int var; };

// Recognise the tcgen05 conv structure and fill its configuration.
bool tc_conv_plan(const GeneralWorkload& w, const Program& p, const Stmt* s, const Expr* xl, const Expr* yl,
                  const std::vector<LoopPart>& lps, bool guarded, const DeviceLimits& lim, TcConvCfg* out) {
  (void)guarded;
  if (xl->kids.size() != 4 || lps.size() < 4) return false;
  const size_t nv = p.vars.size();
  // per X dim affine coefficients (n, h, w, c)
  std::vector<int64_t> xd[4];
  int64_t x0[4];
  for (int d = 0; d < 4; ++d)
    if (!affine_coeffs(xl->kids[static_cast<size_t>(d)], nv, &xd[d], &x0[d])) return false;
  // merge adjacent parts of one axis (innermost coefficients describe the merged loop)
  struct MP { int axis, group; int64_t ext; int var; };
  std::vector<MP> mp;
  for (const LoopPart& q : lps) {
    int g = w.axis_group[static_cast<size_t>(q.axis)];
    if (!mp.empty() && mp.back().axis == q.axis) { mp.back().ext *= q.ext; mp.back().var = q.var; }
    else mp.push_back(MP{q.axis, g, q.ext, q.var});
  }
  const size_t m = mp.size();
  if (m < 4) return false;
  const MP &ph = mp[m - 4], &pw = mp[m - 3], &pn = mp[m - 2], &pk = mp[m - 1];
  auto co = [&](int d, int var) { return xd[d][static_cast<size_t>(var)]; };
  if (ph.group != AG_M || pw.group != AG_M || pn.group != AG_N || pk.group != AG_K) return false;
  if (ph.ext != 8 || pw.ext != 8 || pk.ext != 64 || pn.ext % 16 != 0) return false;
  if (co(1, ph.var) != 1 || co(0, ph.var) || co(2, ph.var) || co(3, ph.var)) return false;
  if (co(2, pw.var) != 1 || co(0, pw.var) || co(1, pw.var) || co(3, pw.var)) return false;
  if (co(3, pk.var) != 1 || co(0, pk.var) || co(1, pk.var) || co(2, pk.var)) return false;
  // Y: N must be the last (contiguous) dim of the weight so a K-major copy exists
  const Buffer& YB = p.buffers[static_cast<size_t>(yl->buffer)];
  const int64_t ncols = YB.shape.back();
  std::vector<int64_t> ystr(YB.shape.size(), 1);
  for (size_t d = YB.shape.size(); d-- > 1;) ystr[d - 1] = ystr[d] * YB.shape[d];
  std::vector<int64_t> cy(nv, 0), cc(nv, 0);
  int64_t y0 = 0, c0 = 0;
  for (size_t d = 0; d < yl->kids.size(); ++d) {
    std::vector<int64_t> c;
    int64_t k0;
    if (!affine_coeffs(yl->kids[d], nv, &c, &k0)) return false;
    for (size_t x = 0; x < nv; ++x) cy[x] += ystr[d] * c[x];
    y0 += ystr[d] * k0;
  }
  const Buffer& CB = p.buffers[static_cast<size_t>(s->buffer)];
  std::vector<int64_t> cstr(CB.shape.size(), 1);
  for (size_t d = CB.shape.size(); d-- > 1;) cstr[d - 1] = cstr[d] * CB.shape[d];
  for (size_t d = 0; d < s->indices.size(); ++d) {
    std::vector<int64_t> c;
    int64_t k0;
    if (!affine_coeffs(s->indices[d], nv, &c, &k0)) return false;
    for (size_t x = 0; x < nv; ++x) cc[x] += cstr[d] * c[x];
    c0 += cstr[d] * k0;
  }
  if (y0 != 0 || cy[static_cast<size_t>(pn.var)] != 1 || cc[static_cast<size_t>(pn.var)] != 1) return false;
  if (cy[static_cast<size_t>(pk.var)] != ncols || cc[static_cast<size_t>(pk.var)] != 0) return false;
  if (cy[static_cast<size_t>(ph.var)] || cy[static_cast<size_t>(pw.var)]) return false;
  for (int d = 0; d < 4; ++d)
    if (co(d, pn.var)) return false;
  TcConvCfg& t = *out;
  std::memset(&t, 0, sizeof t);
  t.x_n0 = x0[0]; t.x_h0 = x0[1]; t.x_w0 = x0[2]; t.x_c0 = x0[3];
  t.c0 = c0;
  t.cc_h1 = cc[static_cast<size_t>(ph.var)];
  t.cc_w1 = cc[static_cast<size_t>(pw.var)];
  t.bn = pn.ext;
  t.splits = t.kt = t.grid_m = t.grid_n = 1;
  bool before_spatial = true;
  // outer loops (everything but the four innermost merged parts)
  size_t outer_loops = lps.size();
  {
    // count loops belonging to the innermost 4 merged parts
    size_t inner = 0;
    int last_axis = -1;
    int merged = 0;
    for (size_t i = lps.size(); i-- > 0;) {
      if (lps[i].axis != last_axis) { ++merged; last_axis = lps[i].axis; }
      if (merged > 4) break;
      ++inner;
    }
    outer_loops = lps.size() - inner;
  }
  for (size_t i = 0; i < outer_loops; ++i) {
    const LoopPart& q = lps[i];
    const size_t v = static_cast<size_t>(q.var);
    int g = w.axis_group[static_cast<size_t>(q.axis)];
    CList* L;
    if (g == AG_K) {
      L = before_spatial ? &t.k_split : &t.k_tile;
      (before_spatial ? t.splits : t.kt) *= q.ext;
    } else {
      before_spatial = false;
      if (g == AG_M) { L = &t.m_grid; t.grid_m *= q.ext; }
      else if (g == AG_N) { L = &t.n_grid; t.grid_n *= q.ext; }
      else return false;
    }
    if (L->n >= 8) return false;
    const int k = L->n++;
    L->ext[k] = q.ext;
    L->xn[k] = xd[0][v];
    L->xh[k] = xd[1][v];
    L->xw[k] = xd[2][v];
    L->xc[k] = xd[3][v];
    if (g == AG_K) {
      if (cy[v] % ncols) return false;
      L->kf[k] = cy[v] / ncols;  // weight row (flattened r, s, ci) of the K-major copy
    } else if (g == AG_N) {
      L->co[k] = cy[v];          // output-channel offset of an N tile
    } else if (cy[v] != 0) {
      return false;
    }
    L->cc[k] = cc[v];
    if (cc[v] % 4) return false;  // float4 epilogue stores
  }
  if (t.c0 % 4 || t.cc_h1 % 4 || t.cc_w1 % 4) return false;
  if (t.splits * t.kt > kConvMaxK) return false;  // per-k-tile coordinate table (tc_conv.cu)
  // fp32 (3xTF32): a ring slot is one 32-channel k sub-tile, hi and lo halves
  // of both operands (twice the bf16 slot), two slots per k-tile; its split-K
  // uses the L2 tickets only (no cluster)
  t.x3 = !lim.bf16;
  const int64_t per_kt = t.x3 ? 2 : 1;
  const int64_t stage = (128 * 64 * 2 + t.bn * 64 * 2) * per_kt;
  const bool cluster = t.splits > 1 && !t.x3;
  const int64_t rows_per = (64 + t.splits - 1) / t.splits;
  const int64_t red = cluster ? t.splits * rows_per * (t.bn + 4) * 4 : 64 * (t.bn + 4) * 4;
  int64_t avail = lim.max_smem - 2048 - (cluster ? red : 0);
  t.stages = std::min<int64_t>(per_kt * t.kt, std::max<int64_t>(1, avail / stage));
  t.stages = std::min<int64_t>(t.stages, 8);
  t.smem_bytes = (cluster ? t.stages * stage + red : std::max(t.stages * stage, red)) + 1024 + 256;
  return true;
}

}  // namespace

// Quasi-affine decomposition of an index expression over the loops of one
// block: sum of coef * ((v_l / div) % mod) terms + constant (generic.hpp).
bool qdecomp(const Expr* e, const std::vector<int>& loop_of_var, int64_t scale, QSum* q);

bool qsingle(const Expr* e, const std::vector<int>& loop_of_var, QTerm* t) {
  QSum tmp;
  if (!qdecomp(e, loop_of_var, 1, &tmp) || tmp.n != 1 || tmp.c0 != 0 || tmp.t[0].coef != 1) return false;
  *t = tmp.t[0];
  return true;
}

bool qdecomp(const Expr* e, const std::vector<int>& loop_of_var, int64_t scale, QSum* q) {
  switch (e->op) {
    case Op::Int: q->c0 += scale * e->value; return true;
    case Op::Var: {
      if (e->var < 0 || static_cast<size_t>(e->var) >= loop_of_var.size() || loop_of_var[e->var] < 0) return false;
      if (q->n == kQMax) return false;
      q->t[q->n++] = QTerm{loop_of_var[e->var], 1, 0, 0, scale};
      return true;
    }
    case Op::Add: return qdecomp(e->kids[0], loop_of_var, scale, q) && qdecomp(e->kids[1], loop_of_var, scale, q);
    case Op::Sub: return qdecomp(e->kids[0], loop_of_var, scale, q) && qdecomp(e->kids[1], loop_of_var, -scale, q);
    case Op::Mul:
      if (e->kids[0]->op == Op::Int) return qdecomp(e->kids[1], loop_of_var, scale * e->kids[0]->value, q);
      if (e->kids[1]->op == Op::Int) return qdecomp(e->kids[0], loop_of_var, scale * e->kids[1]->value, q);
      return false;
    case Op::FloorDiv:
    case Op::Mod: {
      if (e->kids[1]->op != Op::Int || e->kids[1]->value <= 0 || e->kids[1]->value > (1LL << 30)) return false;
      const int64_t k = e->kids[1]->value;
      QTerm t;
      if (!qsingle(e->kids[0], loop_of_var, &t)) return false;
      if (e->op == Op::FloorDiv) {
        if (t.mod && t.mod % k) return false;  // (x % m) / k = (x / k) % (m / k) only when k | m
        if (static_cast<int64_t>(t.div) * k > (1LL << 30)) return false;
        t.div = static_cast<int32_t>(t.div * k);
        if (t.mod) t.mod = static_cast<int32_t>(t.mod / k);
      } else {
        if (t.mod && t.mod % k) return false;  // (x % m) % k = x % k only when k | m
        t.mod = static_cast<int32_t>(k);
      }
      if (q->n == kQMax) return false;
      t.coef = scale;
      q->t[q->n++] = t;
      return true;
    }
    default: return false;
  }
}

// AFFCOPY plan for an elementwise block: value = Load or Select(guard, Load, 0)
// with quasi-affine indices; the guard must be exactly the load's in-bounds
// predicate (checked like SIMT-A's inlined pad, on corners + 256 samples).
bool affcopy_plan(const Program& p, const Block& blk, CopyCfg* c) {
  const Stmt* s = blk.stmt;
  if (s->init || s->epilogue || blk.loops.empty() || static_cast<int>(blk.loops.size()) > kCopyMaxLoops) return false;
  const Expr* xl = nullptr;
  const Expr* cond = nullptr;
  if (!x_side(s->value, &xl, &cond) || xl->buffer == s->buffer) return false;
  std::vector<int> loop_of_var(p.vars.size(), -1);
  c->nl = static_cast<int>(blk.loops.size());
  c->points = 1;
  for (int l = 0; l < c->nl; ++l) {
    const Stmt* L = blk.loops[static_cast<size_t>(l)];
    if (L->var < 0 || static_cast<size_t>(L->var) >= loop_of_var.size()) return false;
    loop_of_var[static_cast<size_t>(L->var)] = l;
    c->ext[l] = L->extent;
    c->points *= L->extent;
  }
  auto strides_of = [&](int buf) {
    const Buffer& B = p.buffers[static_cast<size_t>(buf)];
    std::vector<int64_t> st(B.shape.size(), 1);
    for (size_t d = B.shape.size(); d-- > 1;) st[d - 1] = st[d] * B.shape[d];
    return st;
  };
  auto lin = [&](const std::vector<Expr*>& idx, int buf, QSum* q) {
    std::vector<int64_t> st = strides_of(buf);
    *q = QSum();
    for (size_t d = 0; d < idx.size(); ++d)
      if (!qdecomp(idx[d], loop_of_var, st[d], q)) return false;
    return true;
  };
  if (!lin(s->indices, s->buffer, &c->out) || !lin(xl->kids, xl->buffer, &c->in)) return false;
  // the kernel computes points, offsets and guard values in 32 bits
  auto elems = [&](int buf) {
    int64_t n = 1;
    for (int64_t d : p.buffers[static_cast<size_t>(buf)].shape) n *= d;
    return n;
  };
  if (c->points >= (1LL << 31) || elems(s->buffer) >= (1LL << 30) || elems(xl->buffer) >= (1LL << 30)) return false;
  auto small = [](const QSum& q) {
    if (q.c0 >= (1LL << 30) || q.c0 <= -(1LL << 30)) return false;
    for (int i = 0; i < q.n; ++i)
      if (q.t[i].coef >= (1LL << 30) || q.t[i].coef <= -(1LL << 30)) return false;
    return true;
  };
  if (!small(c->out) || !small(c->in)) return false;
  c->in_buf = xl->buffer;
  c->out_buf = s->buffer;
  // guarded dims: with a Select guard every input dim is checked (cheap);
  // without one the load must be in bounds everywhere (host-sampled below)
  const Buffer& XB = p.buffers[static_cast<size_t>(xl->buffer)];
  c->ng = 0;
  if (cond) {
    if (xl->kids.size() > static_cast<size_t>(kCopyMaxGuard)) return false;
    for (size_t d = 0; d < xl->kids.size(); ++d) {
      c->g[c->ng] = QSum();
      if (!qdecomp(xl->kids[d], loop_of_var, 1, &c->g[c->ng])) return false;
      c->gext[c->ng] = XB.shape[d];
      ++c->ng;
    }
  }
  // contiguous innermost run: loop l joins when its only term in both the
  // input and the output offsets is a plain `coef * v_l` with coef == run so
  // far, and no guard looks at it
  {
    auto only_plain = [](const QSum& q, int l, int64_t want) {
      int found = 0;
      for (int i = 0; i < q.n; ++i)
        if (q.t[i].loop == l) {
          if (q.t[i].div != 1 || q.t[i].mod != 0 || q.t[i].coef != want) return false;
          ++found;
        }
      return found == 1;
    };
    auto absent = [](const QSum& q, int l) {
      for (int i = 0; i < q.n; ++i)
        if (q.t[i].loop == l) return false;
      return true;
    };
    c->run_loops = 0;
    c->run = 1;
    for (int l = c->nl - 1; l >= 0; --l) {
      bool ok = only_plain(c->in, l, c->run) && only_plain(c->out, l, c->run);
      for (int d = 0; d < c->ng && ok; ++d) ok = absent(c->g[d], l);
      if (!ok) break;
      c->run *= c->ext[l];
      ++c->run_loops;
    }
    c->vec = 1;
    for (int v : {8, 4, 2})
      if (c->run % v == 0) { c->vec = v; break; }
  }
  // host check on corners + 256 samples: the guard is exactly the load's
  // in-bounds predicate, and an unguarded load never leaves its buffer
  std::mt19937_64 rng(777);
  std::vector<int64_t> vals(p.vars.size(), 0);
  for (int t = 0; t < 258; ++t) {
    for (const Stmt* L : blk.loops)
      vals[static_cast<size_t>(L->var)] =
          t == 0 ? 0 : t == 1 ? L->extent - 1 : static_cast<int64_t>(rng() % static_cast<uint64_t>(L->extent));
    bool ok = true;
    bool inb = true;
    for (size_t d = 0; d < xl->kids.size(); ++d) {
      int64_t x = host_eval(xl->kids[d], vals, &ok);
      inb &= x >= 0 && x < XB.shape[d];
    }
    if (!ok) return false;
    if (cond) {
      int64_t cv = host_eval(cond, vals, &ok);
      if (!ok || ((cv != 0) != inb)) return false;
    } else if (!inb) {
      return false;
    }
  }
  return true;
}

GeneralPlan plan_general(const GeneralWorkload& w, const Program& p, const DeviceLimits& lim) {
  GeneralPlan plan;
  std::string err;
  if (!encode_generic(p, &plan.gen, &err)) return unsupported("program is not executable by the generic executor");
  for (const Buffer& B : p.buffers) plan.buf_names.push_back(B.name);
  for (const std::string& n : plan.buf_names)
    if (std::find(w.buffers.begin(), w.buffers.end(), n) == w.buffers.end())
      return unsupported("candidate introduces a buffer the workload does not have");
  std::vector<Block> blocks = blocks_preorder(p);
  bool seen_con = false;
  for (size_t bi = 0; bi < blocks.size(); ++bi) {
    const Block& blk = blocks[bi];
    const Stmt* s = blk.stmt;
    GStep step;
    step.block = static_cast<int>(bi);
    if (!s->init) {
      step.family = affcopy_plan(p, blk, &step.copy) ? F_AFFCOPY : F_GENERIC;
      plan.steps.push_back(step);
      continue;
    }
    if (s->name != w.block || seen_con) return unsupported("unexpected reduction block");
    seen_con = true;
    const Expr* v = s->value;
    if (v->op != Op::Mul) return unsupported("contraction value changed shape");
    const Expr* yl = nullptr;
    const Expr* xf = nullptr;
    for (int i = 0; i < 2; ++i)
      if (v->kids[i]->op == Op::Load && p.buffers[static_cast<size_t>(v->kids[i]->buffer)].name == w.y_buf) {
        yl = v->kids[i];
        xf = v->kids[1 - i];
      }
    const Expr* xl = nullptr;
    const Expr* cond = nullptr;
    if (!yl || !x_side(xf, &xl, &cond)) return unsupported("contraction operands changed shape");

    // PVU-scheduled contraction (possibly fused loops): generic nest kernel
    bool block_serial = true;
    for (const Stmt* l : blk.loops) block_serial &= l->kind == Kind::Serial;
    if (!block_serial) {
      if (blk.loops.empty() || blk.loops[0]->kind != Kind::Parallel)
        return unsupported("parallel loop is not outermost");
      step.family = F_NESTGEN;
      plan.family = F_NESTGEN;
      plan.cfg[0] = static_cast<int32_t>(blk.loops[0]->extent);
      plan.steps.push_back(step);
      if (s->epilogue) {
        GStep e = step;
        e.family = F_GENERIC;
        e.epilogue_pass = true;
        plan.steps.push_back(e);
      }
      continue;
    }

    // per-loop axis and stride from the witness expressions
    const size_t nv = p.vars.size();
    const size_t na = w.axis_var.size();
    std::vector<std::vector<int64_t>> coef(na);
    for (size_t a = 0; a < na; ++a) {
      const std::vector<Expr*>* idx = w.wit_buf[a] == "store" ? &s->indices
                                    : w.wit_buf[a] == "y" ? &yl->kids : &xl->kids;
      if (static_cast<size_t>(w.wit_dim[a]) >= idx->size()) return unsupported("witness dim missing");
      int64_t c0 = 0;
      if (!affine_coeffs((*idx)[static_cast<size_t>(w.wit_dim[a])], nv, &coef[a], &c0) || c0 != 0)
        return unsupported("non-affine index (fused loop) in the contraction");
    }
    using LP = LoopPart;
    std::vector<LP> lps;
    for (const Stmt* l : blk.loops) {
      int axis = -1;
      int64_t stride = 0;
      for (size_t a = 0; a < na; ++a) {
        if (coef[a][static_cast<size_t>(l->var)] == 0) continue;
        if (axis >= 0) { axis = -2; break; }
        axis = static_cast<int>(a);
        stride = coef[a][static_cast<size_t>(l->var)];
      }
      if (axis == -2) return unsupported("loop variable feeds two axes");
      if (axis < 0) {
        if (l->extent == 1) continue;
        return unsupported("loop variable unused by the contraction");
      }
      lps.push_back(LP{axis, l->extent, stride, l->kind, l->var});
    }
    bool any_parallel = false, all_serial = true;
    for (const LP& q : lps) {
      all_serial &= q.kind == Kind::Serial;
      any_parallel |= q.kind == Kind::Parallel;
    }
    if (!all_serial) {
      // PVU: the outermost loop of the block must be the parallel one
      if (blk.loops.empty() || blk.loops[0]->kind != Kind::Parallel || !any_parallel)
        return unsupported("parallel loop is not outermost");
      step.family = F_NESTGEN;
      plan.family = F_NESTGEN;
      plan.cfg[0] = static_cast<int32_t>(blk.loops[0]->extent);
      plan.steps.push_back(step);
      if (s->epilogue) {
        GStep e = step;
        e.family = F_GENERIC;
        e.epilogue_pass = true;
        plan.steps.push_back(e);
      }
      continue;
    }
    for (size_t a = 0; a < na; ++a) {
      int64_t inner = 1;
      for (size_t i = lps.size(); i-- > 0;) {
        if (lps[i].axis != static_cast<int>(a)) continue;
        if (lps[i].stride != inner) return unsupported("axis parts not in split order");
        inner *= lps[i].ext;
      }
      if (inner != w.axis_extent[a]) return unsupported("axis parts do not cover the axis");
    }
    std::vector<int> nparts(na, 0);
    for (const LP& q : lps) nparts[static_cast<size_t>(q.axis)]++;
    bool naive = true;
    for (int c : nparts) naive &= c <= 1;
    if (naive) {
      step.family = F_GENERIC;
      plan.family = F_NAIVE;
      plan.steps.push_back(step);
      if (s->epilogue) {
        GStep e = step;
        e.epilogue_pass = true;
        plan.steps.push_back(e);
      }
      continue;
    }
    for (int g : w.axis_group)
      if (g == AG_B) return unsupported("batch axes are instantiated by the SIMT family of single-axis workloads");

    // ---- SIMT-A: address coefficients per loop ----
    AffineCfg& A = step.aff;
    std::memset(&A, 0, sizeof A);
    auto strides_of = [&](int buf) {
      const Buffer& B = p.buffers[static_cast<size_t>(buf)];
      std::vector<int64_t> st(B.shape.size(), 1);
      for (size_t d = B.shape.size(); d-- > 1;) st[d - 1] = st[d] * B.shape[d];
      return st;
    };
    auto lin = [&](const std::vector<Expr*>& idx, int buf, std::vector<int64_t>* per_var, int64_t* c0) {
      std::vector<int64_t> st = strides_of(buf);
      per_var->assign(nv, 0);
      *c0 = 0;
      for (size_t d = 0; d < idx.size(); ++d) {
        std::vector<int64_t> c;
        int64_t k0;
        if (!affine_coeffs(idx[d], nv, &c, &k0)) return false;
        for (size_t x = 0; x < nv; ++x) (*per_var)[x] += st[d] * c[x];
        *c0 += st[d] * k0;
      }
      return true;
    };
    std::vector<int64_t> cx, cy, cc;
    if (!lin(xl->kids, xl->buffer, &cx, &A.x0) || !lin(yl->kids, yl->buffer, &cy, &A.y0) ||
        !lin(s->indices, s->buffer, &cc, &A.c0))
      return unsupported("non-affine operand index");
    // guarded X dims (inlined pad): dims whose index range leaves the buffer
    std::vector<int> gdims;
    std::vector<std::vector<int64_t>> gcoef;
    std::vector<int64_t> gconst;
    const Buffer& XB = p.buffers[static_cast<size_t>(xl->buffer)];
    for (size_t d = 0; d < xl->kids.size(); ++d) {
      std::vector<int64_t> c;
      int64_t k0;
      affine_coeffs(xl->kids[d], nv, &c, &k0);
      int64_t lo = k0, hi = k0;
      for (const LP& q : lps) {
        int64_t t = c[static_cast<size_t>(q.var)] * (q.ext - 1);
        if (t < 0) lo += t; else hi += t;
      }
      if (lo < 0 || hi >= XB.shape[d]) {
        if (!cond) return unsupported("operand index leaves its buffer");
        gdims.push_back(static_cast<int>(d));
        gcoef.push_back(c);
        gconst.push_back(k0);
      }
    }
    if (gdims.size() > 2) return unsupported("more than two guarded dims");
    if (cond) {
      // the Select guard must be exactly the in-bounds predicate of the load:
      // checked on the corners and a deterministic sample of the iteration space
      std::mt19937_64 rng(12345);
      std::vector<int64_t> vals(nv, 0);
      for (int t = 0; t < 256; ++t) {
        for (const LP& q : lps) {
          int64_t x = t == 0 ? 0 : t == 1 ? q.ext - 1 : static_cast<int64_t>(rng() % static_cast<uint64_t>(q.ext));
          vals[static_cast<size_t>(q.var)] = x;
        }
        bool ok = true;
        int64_t cv = host_eval(cond, vals, &ok);
        bool inb = true;
        for (size_t d = 0; d < xl->kids.size(); ++d) {
          int64_t x = host_eval(xl->kids[d], vals, &ok);
          inb &= x >= 0 && x < XB.shape[d];
        }
        if (!ok || ((cv != 0) != inb)) return unsupported("Select guard is not the load's in-bounds predicate");
      }
    }
    // ---- TCGEN05 conv: innermost [p 8][q 8][co BN][ci 64] (bf16) ----
    // fp32: the 3xTF32 tile reads operand halves; the runner splits a
    // workload input once and an in-candidate activation (a pad stage's
    // output) on every launch, right before the conv step
    if ((lim.bf16 || lim.tf32x3) && tc_conv_plan(w, p, s, xl, yl, lps, cond != nullptr, lim, &step.conv)) {
      step.x3_split = step.conv.x3 && p.buffers[static_cast<size_t>(xl->buffer)].role != 0;
      step.family = F_TCCONV;
      step.x_buf = xl->buffer;
      step.y_buf = yl->buffer;
      step.c_buf = s->buffer;
      plan.family = F_TCCONV;
      const TcConvCfg& t = step.conv;
      int32_t* o = plan.cfg;
      o[0] = static_cast<int32_t>(t.grid_m); o[1] = static_cast<int32_t>(t.grid_n);
      o[2] = static_cast<int32_t>(t.bn); o[3] = static_cast<int32_t>(t.splits);
      o[4] = static_cast<int32_t>(t.kt); o[5] = static_cast<int32_t>(t.stages);
      o[6] = static_cast<int32_t>(t.smem_bytes / 1024);
      o[7] = t.x3 ? 1 : 0;
      plan.steps.push_back(step);
      if (t.bn > 256 || t.splits > 16) { plan.status = P_ILLEGAL; plan.why = "conv tile beyond tcgen05 limits"; return plan; }
      if (t.smem_bytes > lim.max_smem) { plan.status = P_ILLEGAL; plan.why = "smem above limit"; return plan; }
      if (s->epilogue) {
        GStep e;
        e.family = F_GENERIC;
        e.block = static_cast<int>(bi);
        e.epilogue_pass = true;
        plan.steps.push_back(e);
      }
      continue;
    }

    A.ng = static_cast<int>(gdims.size());
    for (int g = 0; g < A.ng; ++g) {
      A.g0[g] = gconst[static_cast<size_t>(g)];
      A.gext[g] = XB.shape[static_cast<size_t>(gdims[static_cast<size_t>(g)])];
    }
    // levels: spatial band 0 grid, 1 threads, >= 2 registers; K last part BK
    std::vector<int> band(na, 0), seenk(na, 0);
    if (lps.size() > static_cast<size_t>(kAMaxParts)) return unsupported("too many loops");
    A.nparts = static_cast<int>(lps.size());
    A.gm = A.gn = A.tm = A.tn = A.rm = A.rn = A.bk = A.kt = 1;
    for (size_t i = 0; i < lps.size(); ++i) {
      const LP& q = lps[i];
      APart& P = A.parts[i];
      P.extent = q.ext;
      P.group = w.axis_group[static_cast<size_t>(q.axis)];
      P.cx = cx[static_cast<size_t>(q.var)];
      P.cy = cy[static_cast<size_t>(q.var)];
      P.cc = cc[static_cast<size_t>(q.var)];
      for (int g = 0; g < A.ng; ++g) P.cg[g] = gcoef[static_cast<size_t>(g)][static_cast<size_t>(q.var)];
      if (P.group == AG_K) {
        int idx = ++seenk[static_cast<size_t>(q.axis)];
        P.level = idx == nparts[static_cast<size_t>(q.axis)] ? AL_BK : AL_KTILE;
        if (P.level == AL_BK) A.bk *= q.ext; else A.kt *= q.ext;
      } else {
        int b = band[static_cast<size_t>(q.axis)]++;
        P.level = b == 0 ? AL_GRID : b == 1 ? AL_THREAD : AL_REG;
        int64_t& grid = P.group == AG_M ? A.gm : A.gn;
        int64_t& thr = P.group == AG_M ? A.tm : A.tn;
        int64_t& reg = P.group == AG_M ? A.rm : A.rn;
        (P.level == AL_GRID ? grid : P.level == AL_THREAD ? thr : reg) *= q.ext;
      }
    }
    const int64_t bm = A.tm * A.rm, bn = A.tn * A.rn;
    A.smem_bytes = A.bk * (bm + 1 + bn + 1) * 4 + 16 + (2 * bm + 2 * A.bk + 2 * bn + 2 * (bm + A.bk)) * 4 + 64;
    step.family = F_SIMTA;
    step.x_buf = xl->buffer;
    step.y_buf = yl->buffer;
    step.c_buf = s->buffer;
    plan.family = F_SIMTA;
    int32_t* o = plan.cfg;
    o[0] = 1; o[1] = static_cast<int32_t>(A.gm); o[2] = static_cast<int32_t>(A.gn);
    o[3] = 1; o[4] = static_cast<int32_t>(A.tm); o[5] = static_cast<int32_t>(A.tn);
    o[6] = 1; o[7] = static_cast<int32_t>(A.rm); o[8] = static_cast<int32_t>(A.rn);
    o[9] = static_cast<int32_t>(A.bk); o[10] = static_cast<int32_t>(A.kt);
    o[11] = static_cast<int32_t>(A.smem_bytes / 1024); o[12] = static_cast<int32_t>(A.tm * A.tn);
    plan.steps.push_back(step);
    if (A.tm * A.tn > lim.max_threads) { plan.status = P_ILLEGAL; plan.why = "threads per CTA above 1024"; return plan; }
    if (!simta_tile_supported(A.rm, A.rn)) { plan.status = P_ILLEGAL; plan.why = "register tile outside the lattice"; return plan; }
    if (A.smem_bytes > lim.max_smem) { plan.status = P_ILLEGAL; plan.why = "shared-memory tile above 227 KB"; return plan; }
    if (A.gm > 65535) { plan.status = P_ILLEGAL; plan.why = "grid too large"; return plan; }
    if (s->epilogue) {
      GStep e;
      e.family = F_GENERIC;
      e.block = static_cast<int>(bi);
      e.epilogue_pass = true;
      plan.steps.push_back(e);
    }
  }
  if (!seen_con) return unsupported("candidate lost its contraction block");
  plan.status = P_OK;
  return plan;
}

}  // namespace lsb
