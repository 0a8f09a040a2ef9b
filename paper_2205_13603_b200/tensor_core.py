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

Decisions (all traced, so search and mutation see them):
  * N: ``split(j, [m/16, 16])`` then ``sample_perfect_tile(j_hi, 2)`` gives
    ``BN = 16 * t`` (tcgen05 N granularity is 16 at M=128); BN > 256 is left to
    the hardware validator.
  * K: ``split(k, [K/64, 64])`` then ``sample_perfect_tile(k_hi, 2)`` gives
    (split-K ways, k-tiles per split); 64 bf16 = one 128-byte swizzle row.
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


def _module_class():
    ls = loopsched()
    ir = ls.ir
    from loopsched.spaces import TransformationModule, _block_stmt, _exclusive_chain

    class _UseTensorCore(TransformationModule):
        name = "use_tensor_core"

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
            roles = _contraction_roles(ir, stmt, loops)
            if roles is None:
                return False
            ext = {l.var: l.extent for l in loops}
            return (ext[roles["m"][0]] % UMMA_M == 0
                    and ext[roles["n"][0]] % N_GRAIN == 0
                    and ext[roles["k"][0]] % BLOCK_K == 0)

        def apply(self, state, block):
            path, stmt = _block_stmt(state, block)
            loops = [l for _, l in ir.enclosing_loops(state.program.root, path)]
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
            state.reorder([ks] + batch + [m0, n0, kt, m1, n1, n16, k64])

    return _UseTensorCore


_CLS = None


def use_tensor_core():
    """Factory mirroring the reference's module factories (`src/spaces.py:311`)."""
    global _CLS
    if _CLS is None:
        _CLS = _module_class()
    return _CLS()


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
            modules.append(use_tensor_core())
        else:
            modules.append(ls.space_from_config({"modules": [entry]}).modules[0])
    return ls.compose(modules)


def b200_space_config() -> dict:
    """Default space + the tcgen05 module (the BERT dense/bmm search space)."""
    return {"modules": [{"mlt": {"structure": "SSRSR"}}, {"auto_inline": {}},
                        {"pvu": {"widths": [4, 8]}}, {"tensor_core": {}}]}


def b200_space():
    return space_from_config(b200_space_config())
