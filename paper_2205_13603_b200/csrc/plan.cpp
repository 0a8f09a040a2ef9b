// Trace-to-kernel instantiator.  See plan.hpp for the mapping convention.
#include <cstdlib>
#include "plan.hpp"

#include <algorithm>

namespace lsb {

namespace {

const int64_t kTiles[] = {1, 2, 3, 4, 6, 8, 12, 16, 24, 32, 48, 64};  // simt_impl.cuh SimtTable

bool fail(std::string* err, const char* m) {
  if (err) *err = m;
  return false;
}

int64_t dim_stride(const Buffer& b, int dim) {
  int64_t s = 1;
  for (size_t d = static_cast<size_t>(dim) + 1; d < b.shape.size(); ++d) s *= b.shape[d];
  return s;
}

int var_dim(const std::vector<Expr*>& idx, int var) {
  int found = -1;
  for (size_t d = 0; d < idx.size(); ++d)
    if (idx[d]->op == Op::Var && idx[d]->var == var) {
      if (found >= 0) return -2;
      found = static_cast<int>(d);
    }
  return found;
}

bool is_zero_const(const Expr* e) { return e && e->op == Op::Int && e->value == 0; }

Plan unsupported(const char* why) {
  Plan p;
  p.status = P_UNSUPPORTED;
  p.why = why;
  return p;
}
Plan illegal(Plan p, const char* why) {
  p.status = P_ILLEGAL;
  p.why = why;
  return p;
}

}  // namespace

int simt_tile_index(int64_t v) {
  for (int i = 0; i < kSimtTiles; ++i)
    if (kTiles[i] == v) return i;
  return -1;
}

bool simt_tile_supported(int64_t rm, int64_t rn) {
  return simt_tile_index(rm) >= 0 && simt_tile_index(rn) >= 0 && rm * rn <= 64;
}

bool analyze_workload(const Program& e0, Workload* w, std::string* err) {
  std::vector<Block> blocks = blocks_preorder(e0);
  if (blocks.size() != 1) return fail(err, "runner workloads are single-block contractions");
  const Stmt* s = blocks[0].stmt;
  if (s->type != SType::Compute || !s->init || s->epilogue) return fail(err, "block is not a reduction");
  if (!is_zero_const(s->init)) return fail(err, "reduction init must be 0");
  const Expr* v = s->value;
  if (v->op != Op::Mul || v->kids[0]->op != Op::Load || v->kids[1]->op != Op::Load)
    return fail(err, "block value is not a product of two loads");
  const Expr* X = v->kids[0];
  const Expr* Y = v->kids[1];
  for (const auto* idx : {&s->indices, &X->kids, &Y->kids})
    for (const Expr* e : *idx)
      if (e->op != Op::Var) return fail(err, "e0 indices must be plain loop variables");
  w->block = s->name;
  w->x_buf = X->buffer;
  w->y_buf = Y->buffer;
  w->c_buf = s->buffer;
  if (w->x_buf == w->y_buf || w->x_buf == w->c_buf || w->y_buf == w->c_buf)
    return fail(err, "operands must be distinct buffers");
  const Buffer& BX = e0.buffers[static_cast<size_t>(w->x_buf)];
  const Buffer& BY = e0.buffers[static_cast<size_t>(w->y_buf)];
  const Buffer& BC = e0.buffers[static_cast<size_t>(w->c_buf)];
  int seen[R_COUNT] = {0};
  for (const Stmt* l : blocks[0].loops) {
    int dc = var_dim(s->indices, l->var), dx = var_dim(X->kids, l->var), dy = var_dim(Y->kids, l->var);
    if (dc == -2 || dx == -2 || dy == -2) return fail(err, "a variable indexes two dims of one buffer");
    int role;
    if (dc >= 0 && dx >= 0 && dy >= 0) role = R_BATCH;
    else if (dc >= 0 && dx >= 0 && dy < 0) role = R_M;
    else if (dc >= 0 && dx < 0 && dy >= 0) role = R_N;
    else if (dc < 0 && dx >= 0 && dy >= 0) role = R_K;
    else return fail(err, "loop variable outside the contraction pattern");
    if (seen[role]++) return fail(err, "more than one loop per role");
    w->extent[role] = l->extent;
    if (dx >= 0) w->sx[role] = dim_stride(BX, dx);
    if (dy >= 0) w->sy[role] = dim_stride(BY, dy);
    if (dc >= 0) w->sc[role] = dim_stride(BC, dc);
    if (role == R_N) { w->wit_buf[role] = w->c_buf; w->wit_dim[role] = dc; }
    else { w->wit_buf[role] = w->x_buf; w->wit_dim[role] = dx; }
    if (role == R_K) {
      w->x_kmajor = dx == static_cast<int>(BX.shape.size()) - 1;
      w->y_kmajor = dy == static_cast<int>(BY.shape.size()) - 1;
    }
  }
  if (!seen[R_M] || !seen[R_N] || !seen[R_K]) return fail(err, "need one M, N and K loop");
  w->has_batch = seen[R_BATCH] != 0;
  w->input_bufs.clear();
  for (size_t b = 0; b < e0.buffers.size(); ++b)
    if (e0.buffers[b].role == 0) w->input_bufs.push_back(static_cast<int>(b));
  auto elems = [](const Buffer& b) { int64_t n = 1; for (int64_t x : b.shape) n *= x; return n; };
  w->x_elems = elems(BX);
  w->y_elems = elems(BY);
  w->c_elems = elems(BC);
  return true;
}

Plan plan_program(const Workload& w, const Program& p, const DeviceLimits& lim) {
  std::vector<Block> blocks = blocks_preorder(p);
  if (blocks.size() != 1) return unsupported("multi-block program");
  const Block& blk = blocks[0];
  const Stmt* s = blk.stmt;
  if (s->type != SType::Compute) return unsupported("tensorized block (tu.mma4) has no B200 mapping");
  if (s->name != w.block || !s->init || s->epilogue) return unsupported("block does not match the workload");
  const Expr* v = s->value;
  if (v->op != Op::Mul || v->kids[0]->op != Op::Load || v->kids[1]->op != Op::Load)
    return unsupported("block value changed shape");
  const Expr* X = v->kids[0]->buffer == w.x_buf ? v->kids[0] : v->kids[1];
  const Expr* Y = X == v->kids[0] ? v->kids[1] : v->kids[0];
  if (X->buffer != w.x_buf || Y->buffer != w.y_buf || s->buffer != w.c_buf)
    return unsupported("operand buffers changed");

  // role index expressions -> per-loop (role, stride)
  const size_t nv = p.vars.size();
  std::vector<std::vector<int64_t>> coeff(R_COUNT);
  for (int r = 0; r < R_COUNT; ++r) {
    if (r == R_BATCH && !w.has_batch) continue;
    const Expr* e = nullptr;
    if (w.wit_buf[r] == w.c_buf) e = s->indices[static_cast<size_t>(w.wit_dim[r])];
    else e = X->kids[static_cast<size_t>(w.wit_dim[r])];
    int64_t c0 = 0;
    if (!affine_coeffs(e, nv, &coeff[r], &c0) || c0 != 0)
      return unsupported("non-affine index (fused loop) in the contraction");
  }
  std::vector<Part> parts;
  for (const Stmt* l : blk.loops) {
    int role = -1;
    int64_t stride = 0;
    for (int r = 0; r < R_COUNT; ++r) {
      if (coeff[r].empty() || coeff[r][static_cast<size_t>(l->var)] == 0) continue;
      if (role >= 0) return unsupported("loop variable feeds two axes");
      role = r;
      stride = coeff[r][static_cast<size_t>(l->var)];
    }
    if (role < 0) {
      if (l->extent == 1) continue;
      return unsupported("loop variable unused by the contraction");
    }
    if (stride <= 0) return unsupported("negative stride");
    parts.push_back(Part{role, l->extent, stride, l->kind});
  }
  // canonical split order per axis: strides are the mixed radix of the
  // extents inside, outermost first (`split` recombination, src/schedule.py:290-295)
  for (int r = 0; r < R_COUNT; ++r) {
    int64_t inner = 1;
    for (size_t i = parts.size(); i-- > 0;) {
      if (parts[i].role != r) continue;
      if (parts[i].stride != inner) return unsupported("axis parts not in split order");
      inner *= parts[i].extent;
    }
    if (inner != w.extent[r]) return unsupported("axis parts do not cover the axis");
  }
  Plan plan;
  plan.status = P_OK;
  bool all_serial = true;
  for (const Part& q : parts) all_serial &= q.kind == Kind::Serial;
  // traced pipeline depth (tensor_core.py, pipeline=True): the only
  // non-serial loop is an unrolled K part directly above the tile's M part;
  // it is a k-tile loop like any other, its extent the stage count
  int64_t traced_stages = 0;
  {
    int nonserial = 0;
    size_t at = 0;
    for (size_t i = 0; i < parts.size(); ++i)
      if (parts[i].kind != Kind::Serial) {
        ++nonserial;
        at = i;
      }
    if (nonserial == 1 && (lim.bf16 || lim.tf32x3) && parts[at].kind == Kind::Unrolled && parts[at].role == R_K &&
        at + 1 < parts.size() && parts[at + 1].role == R_M) {
      traced_stages = parts[at].extent;
      parts[at].kind = Kind::Serial;
      all_serial = true;
    }
  }

  if (!all_serial) {
    // LOOPNEST: parallel outermost loop -> threads; everything else in order
    if (parts.empty() || parts[0].kind != Kind::Parallel) return unsupported("parallel loop is not outermost");
    if (parts.size() > static_cast<size_t>(kMaxLoopNest)) return unsupported("loop nest too deep");
    plan.family = F_LOOPNEST;
    plan.parts = parts;
    plan.nest.n = static_cast<int>(parts.size());
    for (size_t i = 0; i < parts.size(); ++i) {
      const Part& q = parts[i];
      plan.nest.ext[i] = q.extent;
      plan.nest.dx[i] = q.stride * w.sx[q.role];
      plan.nest.dy[i] = q.stride * w.sy[q.role];
      plan.nest.dc[i] = q.stride * w.sc[q.role];
    }
    plan.needs_zero = true;
    plan.cfg[0] = static_cast<int32_t>(parts[0].extent);
    plan.cfg[1] = static_cast<int32_t>(parts.size());
    return plan;
  }

  // merge adjacent parts of one axis (identical iteration order)
  std::vector<Part> merged;
  for (const Part& q : parts) {
    if (!merged.empty() && merged.back().role == q.role) {
      merged.back().extent *= q.extent;
      merged.back().stride = q.stride;
    } else {
      merged.push_back(q);
    }
  }
  plan.parts = merged;
  int nparts[R_COUNT] = {0};
  for (const Part& q : merged) nparts[q.role]++;

  bool naive = true;
  for (int r = 0; r < R_COUNT; ++r) naive &= nparts[r] <= 1;
  if (naive) {
    plan.family = F_NAIVE;
    plan.cfg[0] = 256;
    return plan;
  }

  // ---- TCGEN05: innermost [M 128][N BN][K 64] tile --------------------------
  size_t np = merged.size();
  if ((lim.bf16 || lim.tf32x3) && np >= 3) {
    const Part& pm = merged[np - 3];
    const Part& pn = merged[np - 2];
    const Part& pk = merged[np - 1];
    if (pm.role == R_M && pn.role == R_N && pk.role == R_K && pm.extent == 128 && pk.extent == 64 &&
        pn.extent % 16 == 0) {
      plan.family = F_TC;
      TcCfg& t = plan.tc;
      t.bn = pn.extent;
      t.batch = w.extent[R_BATCH];
      t.grid_m = w.extent[R_M] / 128;
      t.grid_n = w.extent[R_N] / t.bn;
      t.splits = 1;
      t.kt = 1;
      t.x3 = !lim.bf16;
      bool before_spatial = true;
      for (size_t i = 0; i + 3 < np; ++i) {
        if (merged[i].role != R_K) { before_spatial = false; continue; }
        if (before_spatial) t.splits *= merged[i].extent;
        else t.kt *= merged[i].extent;
      }
      // stage count: the traced pipeline depth, or as many k-tiles as fit in
      // shared memory (<= 8)
      const int64_t tiles = t.batch * t.grid_m * t.grid_n;
      // (3xTF32 ring slots are 32-element k sub-tiles: two per k-tile)
      const int64_t per_kt = t.x3 ? 2 : 1;
      const TcGeom g0 = tc_geom(t.bn, t.splits, 1, tiles, t.x3);
      const int64_t avail = lim.max_smem - 1024 - 256;
      const int64_t fit = std::max<int64_t>(1, avail / g0.stage_bytes);
      const int64_t slots = per_kt * t.kt;
      t.stages = traced_stages ? std::min(per_kt * traced_stages, slots) : std::min<int64_t>({slots, fit, 8});
      if (per_kt * traced_stages > fit) return illegal(plan, "traced pipeline depth above shared memory");
      const TcGeom g = tc_geom(t.bn, t.splits, t.stages, tiles, t.x3);
      plan.needs_zero = g.mode == 3;
      t.smem_bytes = g.smem;
      int32_t* c = plan.cfg;
      c[0] = static_cast<int32_t>(t.batch); c[1] = static_cast<int32_t>(t.grid_m);
      c[2] = static_cast<int32_t>(t.grid_n); c[3] = static_cast<int32_t>(t.bn);
      c[4] = static_cast<int32_t>(t.splits); c[5] = static_cast<int32_t>(t.kt);
      c[6] = static_cast<int32_t>(t.stages); c[7] = static_cast<int32_t>(t.smem_bytes / 1024);
      c[8] = t.x3 ? 1 : 0;
      if (t.bn > 256) return illegal(plan, "UMMA N above 256");
      if (t.smem_bytes > lim.max_smem) return illegal(plan, "shared-memory ring + reduction buffer above 227 KB");
      if (t.batch * t.splits > 65535 || t.grid_m > 65535) return illegal(plan, "grid too large");
      return plan;
    }
  }

  if (traced_stages) return unsupported("unrolled k-tile loop outside a tcgen05 tile");

  // ---- SIMT: grid / threads / registers per spatial axis ------------------
  plan.family = F_SIMT;
  SimtCfg& c = plan.simt;
  int64_t g[3] = {1, 1, 1}, th[3] = {1, 1, 1}, rg[3] = {1, 1, 1};  // batch, m, n
  int band[R_COUNT] = {0};
  int64_t bk = 1, kt = 1;
  int kparts = nparts[R_K];
  int kseen = 0;
  for (const Part& q : merged) {
    if (q.role == R_K) {
      if (++kseen == kparts) bk = q.extent;
      else kt *= q.extent;
      continue;
    }
    int a = q.role == R_BATCH ? 0 : q.role == R_M ? 1 : 2;
    int b = band[q.role]++;
    if (b == 0) g[a] *= q.extent;
    else if (b == 1) th[a] *= q.extent;
    else rg[a] *= q.extent;
  }
  c.gb = g[0]; c.gm = g[1]; c.gn = g[2];
  c.tb = th[0]; c.tm = th[1]; c.tn = th[2];
  c.rb = rg[0]; c.rm = rg[1]; c.rn = rg[2];
  c.bk = bk; c.kt = kt;
  int64_t bm = c.tm * c.rm, bn = c.tn * c.rn;
  c.smem_bytes = c.tb * c.bk * (bm + bn + 2) * 4 + 16;  // rows padded by up to one word each
  if (c.smem_bytes > lim.max_smem) {
    // a long innermost K part is staged in chunks (k-tiles of a divisor of
    // it, a multiple of 8 when one fits): every thread still sums k in loop
    // order, so the result is bit-identical to staging the part whole
    const int64_t per_k = c.tb * (bm + bn + 2) * 4;
    int64_t best = 0, best8 = 0;
    for (int64_t d = c.bk - 1; d >= 1; --d) {
      if (c.bk % d || per_k * d + 16 > lim.max_smem) continue;
      if (!best) best = d;
      if (d % 8 == 0) { best8 = d; break; }
    }
    const int64_t d = best8 * 2 >= best ? best8 : best;
    if (d) {
      c.kt *= c.bk / d;
      c.bk = d;
      c.smem_bytes = per_k * d + 16;
    }
  }
  int64_t threads = c.tb * c.tm * c.tn;
  int32_t* o = plan.cfg;
  o[0] = static_cast<int32_t>(c.gb); o[1] = static_cast<int32_t>(c.gm); o[2] = static_cast<int32_t>(c.gn);
  o[3] = static_cast<int32_t>(c.tb); o[4] = static_cast<int32_t>(c.tm); o[5] = static_cast<int32_t>(c.tn);
  o[6] = static_cast<int32_t>(c.rb); o[7] = static_cast<int32_t>(c.rm); o[8] = static_cast<int32_t>(c.rn);
  o[9] = static_cast<int32_t>(c.bk); o[10] = static_cast<int32_t>(c.kt);
  o[11] = static_cast<int32_t>(c.smem_bytes / 1024); o[12] = static_cast<int32_t>(threads);
  if (threads > lim.max_threads) return illegal(plan, "threads per CTA above 1024");
  if (!simt_tile_supported(c.rm, c.rn)) return illegal(plan, "register tile outside the compiled lattice");
  if (c.smem_bytes > lim.max_smem) return illegal(plan, "shared-memory tile above 227 KB");
  if (c.gm > 65535 || c.gb > 65535) return illegal(plan, "grid too large");
  return plan;
}

}  // namespace lsb
