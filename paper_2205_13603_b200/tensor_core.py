"""`use_tensor_core`: a transformation module that exposes tcgen05-legal tiles.

It is the B200 analog of the reference's ``_UseTensorUnit``
(`src/spaces.py:255-308`) and plugs in through the same
``TransformationModule`` API (`src/spaces.py:21-40`): analysis in
``applicability``, traced sampling + primitives in ``apply``.  It never adds an
intrinsic: it only splits and reorders, so every program it
produces is still executable by the reference interpreter and priced by the
reference simulator.  The B200 instantiator recognises the resulting nest
structurally: the three innermost loops
``[M 128][N BN][K 64]`` become one tcgen05 tile, the reduction part hoisted
outside every spatial loop becomes split-K, and the remaining spatial parts
become the CTA grid.

NHWC conv2d (implicit GEMM): output pixels are tiled into 8 x 8 boxes (the
M rows of the tile), output channels into BN = 16 * t, input channels into
64-wide k-tiles, and the filter rows r into (split-K ways, in-loop rows):
``[r_split][n][p0][q0][co0][r_in][s][ci0][p 8][q 8][co BN][ci 64]``.

Decisions (all traced, so search and mutation see them):
  * N: ``split(j, [m/16, 16])`` then ``sample_perfect_tile(j_hi, 2)`` gives
    ``BN = 16 * t`` (tcgen05 N granularity is 16 at M=128); BN > 256 is left to
    the hardware validator.
  * K: ``split(k, [K/64, 64])`` then ``sample_perfect_tile(k_hi, 2)`` gives
    (split-K ways, k-tiles per split); 64 bf16 = one 128-byte swizzle row.
  * pipeline depth (``use_tensor_core(pipeline=True)``): the k-tiles of a
    split are split once more, ``sample_perfect_tile(kt, 2)`` -> (kt / S, S),
    and the inner part is ``unroll``-ed; the instantiator reads S as the
    number of shared-memory stages in flight (ILLEGAL above what fits).
"""

from __future__ import annotations

from .refapi import loopsched

UMMA_M = 128
N_GRAIN = 16
BLOCK_K = 64


def _contraction_roles(ir, stmt, loops):
    """(batch, m, n, k) loop-var lists for C[...] += A[...] * B[...] with
    single-variable indices, or None."""
    v = stmt.value
    if not (isinstance(v, ir.BinOp) and v.op == "mul"
            and isinstance(v.a, ir.Load) and isinstance(v.b, ir.Load)):
        return None
    for idx in (stmt.indices, v.a.indices, v.b.indices):
        if not all(isinstance(e, ir.Var) for e in idx):
            return None
    out = {e.name for e in stmt.indices}
    a = {e.name for e in v.a.indices}
    b = {e.name for e in v.b.indices}
    roles = {"batch": [], "m": [], "n": [], "k": []}
    for l in loops:
        x = l.var
        if x in out and x in a and x in b:
            roles["batch"].append(x)
        elif x in out and x in a:
            roles["m"].append(x)
        elif x in out and x in b:
            roles["n"].append(x)
        elif x in a and x in b:
            roles["k"].append(x)
        else:
            return None
    if len(roles["m"]) != 1 or len(roles["n"]) != 1 or len(roles["k"]) != 1:
        return None
    if len(roles["batch"]) > 1:
        return None
    # the A operand must be the one indexed by M (operand order is free)
    return roles


PIX = 8      # output-pixel box edge: 8 x 8 pixels feed the upper 64 rows of a 128-row UMMA tile
CI_TILE = 64  # input channels per k-tile (one 128-byte swizzle row of bf16)


def _conv_roles(ir, stmt, loops):
    """For O[n,p,q,co] += X[n, p+r(+c), q+s(+c), ci] * W[r,s,ci,co] (the NHWC
    implicit GEMM of `workloads.conv2d_nhwc`): var names by role, or None."""
    v = stmt.value
    if not (isinstance(v, ir.BinOp) and v.op == "mul" and isinstance(v.b, ir.Load)):
        return None
    x, w = v.a, v.b
    if isinstance(x, ir.Select) and isinstance(x.then, ir.Load) \
            and isinstance(x.other, ir.IntConst) and x.other.value == 0:
        x = x.then  # pad inlined as a guarded load (zero outside the image)
    if not isinstance(x, ir.Load):
        return None
    if len(stmt.indices) != 4 or len(x.indices) != 4 or len(w.indices) != 4:
        return None
    if not all(isinstance(e, ir.Var) for e in tuple(stmt.indices) + tuple(w.indices)):
        return None
    n, p, q, co = (e.name for e in stmt.indices)
    r, s, ci, co2 = (e.name for e in w.indices)
    if co2 != co:
        return None
    if not (isinstance(x.indices[0], ir.Var) and x.indices[0].name == n
            and isinstance(x.indices[3], ir.Var) and x.indices[3].name == ci):
        return None
    for d, (a, b) in ((1, (p, r)), (2, (q, s))):
        dec = ir.affine_coeffs(x.indices[d])
        if dec is None or dec[0] != {a: 1, b: 1}:
            return None
    names = [l.var for l in loops]
    if sorted(names) != sorted([n, p, q, co, r, s, ci]):
        return None
    return {"n": n, "p": p, "q": q, "co": co, "r": r, "s": s, "ci": ci}


def _module_class():
    ls = loopsched()
    ir = ls.ir
    from loopsched.spaces import TransformationModule, _block_stmt, _exclusive_chain

    class _UseTensorCore(TransformationModule):
        name = "use_tensor_core"

        def __init__(self, pipeline: bool = False):
            self.pipeline = pipeline

        def applicability(self, state, block):
            if not state.block_exists(block):
                return False
            path, stmt = _block_stmt(state, block)
            if not isinstance(stmt, ir.Compute) or stmt.init is None \
                    or stmt.epilogue is not None:
                return False
            if not _exclusive_chain(state, block):
                return False
            loops = [l for _, l in ir.enclosing_loops(state.program.root, path)]
            if any(l.kind != "serial" for l in loops):
                return False
            ext = {l.var: l.extent for l in loops}
            conv = _conv_roles(ir, stmt, loops)
            if conv is not None:
                return (ext[conv["p"]] % PIX == 0 and ext[conv["q"]] % PIX == 0
                        and ext[conv["ci"]] % CI_TILE == 0 and ext[conv["co"]] % N_GRAIN == 0)
            roles = _contraction_roles(ir, stmt, loops)
            if roles is None:
                return False
            return (ext[roles["m"][0]] % UMMA_M == 0
                    and ext[roles["n"][0]] % N_GRAIN == 0
                    and ext[roles["k"][0]] % BLOCK_K == 0)

        def _apply_conv(self, state, block, loops, c):
            refs = state.get_loops(block)
            by_var = {state._resolve_loop(r)[1].var: r for r in refs}
            ext = {l.var: l.extent for l in loops}
            p0, p1 = state.split(by_var[c["p"]], [ext[c["p"]] // PIX, PIX])
            q0, q1 = state.split(by_var[c["q"]], [ext[c["q"]] // PIX, PIX])
            co_hi, co16 = state.split(by_var[c["co"]], [ext[c["co"]] // N_GRAIN, N_GRAIN])
            co0, co1 = state.split(co_hi, state.sample_perfect_tile(co_hi, 2))
            ci0, ci1 = state.split(by_var[c["ci"]], [ext[c["ci"]] // CI_TILE, CI_TILE])
            rs, rt = state.split(by_var[c["r"]], state.sample_perfect_tile(by_var[c["r"]], 2))
            state.reorder([rs, by_var[c["n"]], p0, q0, co0, rt, by_var[c["s"]], ci0, p1, q1, co1, co16, ci1])

        def apply(self, state, block):
            path, stmt = _block_stmt(state, block)
            loops = [l for _, l in ir.enclosing_loops(state.program.root, path)]
            conv = _conv_roles(ir, stmt, loops)
            if conv is not None:
                return self._apply_conv(state, block, loops, conv)
            roles = _contraction_roles(ir, stmt, loops)
            refs = state.get_loops(block)
            by_var = {state._resolve_loop(r)[1].var: r for r in refs}
            ext = {l.var: l.extent for l in loops}
            mv, nv, kv = roles["m"][0], roles["n"][0], roles["k"][0]

            m0, m1 = state.split(by_var[mv], [ext[mv] // UMMA_M, UMMA_M])
            n_hi, n16 = state.split(by_var[nv], [ext[nv] // N_GRAIN, N_GRAIN])
            n0, n1 = state.split(n_hi, state.sample_perfect_tile(n_hi, 2))
            k_hi, k64 = state.split(by_var[kv], [ext[kv] // BLOCK_K, BLOCK_K])
            ks, kt = state.split(k_hi, state.sample_perfect_tile(k_hi, 2))
            batch = [by_var[b] for b in roles["batch"]]
            if self.pipeline:  # traced stage count: the unrolled inner k-tile part
                kto, kst = state.split(kt, state.sample_perfect_tile(kt, 2))
                state.unroll(kst)
                state.reorder([ks] + batch + [m0, n0, kto, kst, m1, n1, n16, k64])
            else:
                state.reorder([ks] + batch + [m0, n0, kt, m1, n1, n16, k64])

    return _UseTensorCore


_CLS = None


def use_tensor_core(pipeline: bool = False):
    """Factory mirroring the reference's module factories (`src/spaces.py:311`)."""
    global _CLS
    if _CLS is None:
        _CLS = _module_class()
    return _CLS(pipeline=pipeline)


def space_from_config(doc: dict):
    """The reference's ``space_from_config`` (`src/spaces.py:478-505`) plus a
    ``{"tensor_core": {}}`` module kind."""
    ls = loopsched()
    if not isinstance(doc, dict) or "modules" not in doc:
        raise ValueError("space config must be an object with a 'modules' list")
    modules = []
    for i, entry in enumerate(doc["modules"]):
        if not isinstance(entry, dict) or len(entry) != 1:
            raise ValueError(f"modules[{i}]: expected a single-key object")
        kind = next(iter(entry))
        if kind == "tensor_core":
            opts = entry[kind] or {}
            modules.append(use_tensor_core(pipeline=bool(opts.get("pipeline", False))))
        else:
            modules.append(ls.space_from_config({"modules": [entry]}).modules[0])
    return ls.compose(modules)


def b200_space_config(pipeline: bool = False) -> dict:
    """Default space + the tcgen05 module (the BERT dense/bmm search space);
    ``pipeline`` adds the traced stage count."""
    return {"modules": [{"mlt": {"structure": "SSRSR"}}, {"auto_inline": {}},
                        {"pvu": {"widths": [4, 8]}},
                        {"tensor_core": {"pipeline": True} if pipeline else {}}]}


def b200_space(pipeline: bool = False):
    return space_from_config(b200_space_config(pipeline))
