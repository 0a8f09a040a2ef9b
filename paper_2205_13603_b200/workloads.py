"""Workload builders the reference lacks: batched matmul and NHWC conv2d.

Both are written against the reference IR (`src/ir.py:109-175`) with the same
conventions as its builders (`src/workloads.py:26-109`): every index is a
plain loop variable (or an affine combination for the convolution window),
padding is materialised by a guarded elementwise stage exactly like
``conv1d``'s pad stage (`src/workloads.py:84-96`), and the result is checked
with ``ir.check_valid``.  SURVEY.md §8a-13 records that both shapes fit the IR
unchanged and that MLT / PVU / auto_inline apply to them.

``batch_matmul`` stores B as ``[batch, n_cols, k]`` (K-major), the layout of
TOPI's ``batch_matmul`` and of attention's ``Q·Kᵀ``.
"""

from __future__ import annotations

from .refapi import loopsched


def batch_matmul(b: int = 12, n: int = 128, m: int = 128, k: int = 64):
    """C[b,i,j] = sum_k A[b,i,k] * B[b,j,k]."""
    ls = loopsched()
    ir = ls.ir
    for name, v in (("b", b), ("n", n), ("m", m), ("k", k)):
        if v < 1:
            raise ValueError(f"{name} must be a positive integer, got {v}")
    body = ir.Compute(
        "bmm", "C", (ir.var("b"), ir.var("i"), ir.var("j")),
        ir.mul(ir.load("A", ir.var("b"), ir.var("i"), ir.var("k")),
               ir.load("B", ir.var("b"), ir.var("j"), ir.var("k"))),
        init=ir.IntConst(0))
    nest = ir.Loop("k", k, "serial", (body,))
    nest = ir.Loop("j", m, "serial", (nest,))
    nest = ir.Loop("i", n, "serial", (nest,))
    nest = ir.Loop("b", b, "serial", (nest,))
    p = ir.TensorProgram(
        buffers=(ir.Buffer("A", (b, n, k), "input"),
                 ir.Buffer("B", (b, m, k), "input"),
                 ir.Buffer("C", (b, n, m), "output")),
        root=(nest,))
    ir.check_valid(p)
    return p


def _inside(ir, x, lo_pad: int, size: int):
    """1 exactly when pad <= x < size + pad (guard arithmetic only, so every
    index stays quasi-affine; mirrors the conv1d guard construction)."""
    lo = ir.emin(ir.emax(ir.add(ir.sub(x, ir.IntConst(lo_pad)), ir.IntConst(1)),
                         ir.IntConst(0)), ir.IntConst(1))
    hi = ir.emin(ir.emax(ir.sub(ir.IntConst(size + lo_pad), x), ir.IntConst(0)),
                 ir.IntConst(1))
    return ir.mul(lo, hi)


def conv2d_nhwc(n: int = 1, h: int = 56, w: int = 56, ci: int = 64, co: int = 64,
                r: int = 3, s: int = 3, stride: int = 1, pad: int = 1):
    """O[n,p,q,co] = sum_{r,s,ci} X[n, p*st+r-pad, q*st+s-pad, ci] * W[r,s,ci,co]
    with the zero padding materialised by a pad stage P (HWIO weights)."""
    ls = loopsched()
    ir = ls.ir
    for name, v in (("n", n), ("h", h), ("w", w), ("ci", ci), ("co", co),
                    ("r", r), ("s", s), ("stride", stride)):
        if v < 1:
            raise ValueError(f"{name} must be a positive integer, got {v}")
    if pad < 0:
        raise ValueError("pad must be non-negative")
    oh_span, ow_span = h + 2 * pad - r, w + 2 * pad - s
    if oh_span < 0 or ow_span < 0 or oh_span % stride or ow_span % stride:
        raise ValueError("conv2d shape mismatch: (size + 2*pad - kernel) must be a "
                         "non-negative multiple of stride")
    oh, ow = oh_span // stride + 1, ow_span // stride + 1
    buffers = [ir.Buffer("X", (n, h, w, ci), "input"),
               ir.Buffer("W", (r, s, ci, co), "input")]
    stmts = []
    src = "X"
    if pad > 0:
        src = "P"
        buffers.append(ir.Buffer("P", (n, h + 2 * pad, w + 2 * pad, ci), "intermediate"))
        yv, xv = ir.var("py"), ir.var("px")
        guard = ir.mul(_inside(ir, yv, pad, h), _inside(ir, xv, pad, w))
        padc = ir.Compute(
            "pad", "P", (ir.var("pn"), yv, xv, ir.var("pc")),
            ir.Select(guard, ir.load("X", ir.var("pn"), ir.sub(yv, ir.IntConst(pad)),
                                     ir.sub(xv, ir.IntConst(pad)), ir.var("pc")),
                      ir.IntConst(0)))
        nest = ir.Loop("pc", ci, "serial", (padc,))
        nest = ir.Loop("px", w + 2 * pad, "serial", (nest,))
        nest = ir.Loop("py", h + 2 * pad, "serial", (nest,))
        stmts.append(ir.Loop("pn", n, "serial", (nest,)))
    buffers.append(ir.Buffer("O", (n, oh, ow, co), "output"))

    def pos(o, k):
        base = ir.var(o) if stride == 1 else ir.mul(ir.var(o), ir.IntConst(stride))
        return ir.add(base, ir.var(k))

    conv = ir.Compute(
        "conv", "O", (ir.var("n"), ir.var("p"), ir.var("q"), ir.var("co")),
        ir.mul(ir.load(src, ir.var("n"), pos("p", "r"), pos("q", "s"), ir.var("ci")),
               ir.load("W", ir.var("r"), ir.var("s"), ir.var("ci"), ir.var("co"))),
        init=ir.IntConst(0))
    nest = ir.Loop("ci", ci, "serial", (conv,))
    nest = ir.Loop("s", s, "serial", (nest,))
    nest = ir.Loop("r", r, "serial", (nest,))
    nest = ir.Loop("co", co, "serial", (nest,))
    nest = ir.Loop("q", ow, "serial", (nest,))
    nest = ir.Loop("p", oh, "serial", (nest,))
    stmts.append(ir.Loop("n", n, "serial", (nest,)))
    prog = ir.TensorProgram(tuple(buffers), tuple(stmts))
    ir.check_valid(prog)
    return prog


def bert_base_tasks(seq: int = 128):
    """The BERT-base (seq 128, batch 1) operator tasks of BASELINE config 5,
    with their per-layer multiplicity."""
    ls = loopsched()
    return [
        ("dense_qkvo", ls.gmm(seq, 768, 768), 4),
        ("ffn_in", ls.gmm(seq, 3072, 768), 1),
        ("ffn_out", ls.gmm(seq, 768, 3072), 1),
        ("attn_qk", batch_matmul(12, seq, seq, 64), 1),
        ("attn_pv", batch_matmul(12, seq, 64, seq), 1),
    ]


BUILDERS = {"batch_matmul": batch_matmul, "conv2d_nhwc": conv2d_nhwc}


def build(name: str, shape=()):
    """Builtin reference workloads plus the two added here."""
    if name in BUILDERS:
        return BUILDERS[name](*[int(s) for s in shape])
    return loopsched().build_workload(name, list(shape) or None)
