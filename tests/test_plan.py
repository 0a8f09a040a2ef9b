"""Host-side instantiator (trace program -> kernel family + config)."""
import json
from collections import Counter

import pytest

from conftest import load_population
from paper_2205_13603_b200 import native


def plan(e0, progs, dtype="bf16"):
    return native.plan_programs(e0, progs, dtype)


def test_e0_maps_to_naive():
    hdr, _ = load_population("bert_ffn")
    r, = plan(hdr["e0"], [hdr["e0"]])
    assert (r["family"], r["status"]) == ("naive", "OK")


def test_population_families_bert_ffn():
    hdr, pop = load_population("bert_ffn")
    res = plan(hdr["e0"], [p["program"] for p in pop[:1024]])
    c = Counter((r["family"], r["status"]) for r in res)
    assert c[("tcgen05", "OK")] > 40
    assert c[("simt", "OK")] > 100
    assert c[("loopnest", "OK")] >= 1
    for r in res:
        if r["family"] == "tcgen05":
            batch, gm, gn, bn, splits, kt, stages, smem_kb = r["cfg"][:8]
            assert gm * 128 == 128 and gn * bn == 768 and splits * kt * 64 == 3072
            assert (r["status"] == "OK") == (bn <= 256)
            assert 1 <= stages <= min(kt, 8)


def test_fp32_tensor_core_tile_is_3xtf32():
    # the same tcgen05 tile on an fp32 workload: 3xTF32 (cfg[8] = 1), same
    # grid / BN / split-K / k-tiles as the bf16 instantiation; its ring slots
    # are 32-element k sub-tiles of twice the bf16 stage bytes
    hdr, pop = load_population("bert_ffn")
    progs = [p["program"] for p in pop[:300]]
    r16 = plan(hdr["e0"], progs)
    r32 = plan(hdr["e0"], progs, dtype="f32")
    n = 0
    for a, b in zip(r16, r32):
        assert (a["family"] == "tcgen05") == (b["family"] == "tcgen05")
        if a["family"] != "tcgen05":
            continue
        if a["status"] == "OK" and b["status"] == "OK":
            assert a["cfg"][:6] == b["cfg"][:6] and a["cfg"][8] == 0 and b["cfg"][8] == 1
            assert 1 <= b["cfg"][6] <= min(2 * b["cfg"][5], 8)
            n += 1
    assert n > 10


def test_simt_mapping_matches_mlt_bands():
    # MLT SSRSR on gmm: i0 j0 | i1 j1 | k0 | i2 j2 | k1 -> grid/threads/registers
    hdr, pop = load_population("gmm512")
    res = plan(hdr["e0"], [p["program"] for p in pop[:200]], dtype="f32")
    for p, r in zip(pop[:200], res):
        if r["family"] != "simt":
            continue
        gb, gm, gn, tb, tm, tn, rb, rm, rn, bk, kt = r["cfg"][:11]
        assert gm * tm * rm == 512 and gn * tn * rn == 512 and bk * kt == 512
        assert (gb, tb, rb) == (1, 1, 1)
        # hardware limits only: threads, register tile (the 2^a 3^b lattice
        # covers every divisor of 512), shared memory after k-chunking
        lattice = (1, 2, 3, 4, 6, 8, 12, 16, 24, 32, 48, 64)
        legal = tm * tn <= 1024 and rm * rn <= 64 and rm in lattice and rn in lattice \
            and bk * (tm * rm + tn * rn + 2) * 4 + 16 <= 227 * 1024
        assert (r["status"] == "OK") == legal, r
        if r["status"] == "OK" and bk > 1:
            assert 512 % bk == 0


def test_bmm_batch_axis_mapping():
    hdr, pop = load_population("bmm_qk")
    res = plan(hdr["e0"], [p["program"] for p in pop[:300]])
    for r in res:
        if r["family"] == "simt" and r["status"] == "OK":
            gb, gm, gn, tb, tm, tn, rb, rm, rn, bk, kt = r["cfg"][:11]
            assert gb * tb * rb == 12 and gm * tm * rm == 128 and gn * tn * rn == 128
        if r["family"] == "tcgen05":
            assert r["cfg"][0] == 12 and r["status"] == "OK"


def test_unsupported_workload_is_reported():
    # an elementwise-only program has no contraction for the runner to time
    relu = ('{"buffers": [{"name": "A", "role": "input", "shape": [8]}, {"name": "B", "role": "output", '
            '"shape": [8]}], "root": [{"loop": {"body": [{"compute": {"buffer": "B", "indices": [{"var": "i"}], '
            '"name": "relu", "value": {"max": [{"load": {"buffer": "A", "indices": [{"var": "i"}]}}, {"int": 0}]}}}], '
            '"extent": 8, "kind": "serial", "var": "i"}}]}')
    with pytest.raises(native.NativeError, match="no contraction block"):
        plan(relu, [relu])


def test_conv2d_general_families():
    hdr, pop = load_population("conv2d")
    res = plan(hdr["e0"], [p["program"] for p in pop])
    fams = Counter((r["family"], r["status"]) for r in res)
    assert fams[("simt_affine", "OK")] > 100 and fams[("nestgen", "OK")] > 0
    assert fams[("tcgen05_conv", "OK")] > 10
    for r in res:
        if r["family"] == "tcgen05_conv":
            gm, gn, bn, splits, kt = r["cfg"][:5]
            assert gm * 64 == 56 * 56 and gn * bn == 64 and splits * kt * 64 == 3 * 3 * 64
        if r["family"] == "simt_affine":
            gb, gm, gn, tb, tm, tn, rb, rm, rn, bk, kt = r["cfg"][:11]
            assert gm * tm * rm == 56 * 56 and gn * tn * rn == 64 and bk * kt == 3 * 3 * 64
    e0r, = plan(hdr["e0"], [hdr["e0"]])
    assert (e0r["family"], e0r["status"]) == ("naive", "OK")


def test_parse_errors_are_per_candidate():
    hdr, pop = load_population("bmm_qk")
    res = plan(hdr["e0"], ["{not json", pop[0]["program"]])
    assert res[0]["status"] == "PARSE"
    assert res[1]["status"] in ("OK", "ILLEGAL")


def test_fused_pvu_schedules_fall_back_to_the_general_families():
    # PVU fuses small leading loops into floordiv / mod indices, which the
    # contraction instantiator cannot map; such candidates run through the
    # general families (NESTGEN) instead of being reported UNSUPPORTED
    import pytest
    from conftest import has_reference
    if not has_reference():
        pytest.skip("reference not importable")
    from paper_2205_13603_b200.refapi import loopsched
    from paper_2205_13603_b200.tensor_core import b200_space
    from paper_2205_13603_b200.workloads import batch_matmul
    ls = loopsched()
    e0 = batch_matmul(3, 33, 17, 24)
    progs = [ls.ir.serialize(p) for p, _ in ls.spaces.sample_traces(e0, b200_space(), 48, seed=7)]
    res = plan(ls.ir.serialize(e0), progs)
    c = Counter((r["family"], r["status"]) for r in res)
    assert c[("nestgen", "OK")] > 0
    assert not [r for r in res if r["status"] == "UNSUPPORTED"]


@pytest.mark.skipif(not __import__("conftest").has_reference(), reason="needs the reference package")
def test_traced_pipeline_depth_sets_tcgen05_stages():
    # use_tensor_core(pipeline=True): the unrolled inner k-tile part is the
    # stage count of the tcgen05 candidate (ILLEGAL above what fits)
    from paper_2205_13603_b200.refapi import loopsched
    from paper_2205_13603_b200.tensor_core import b200_space
    ls = loopsched()
    e0 = ls.gmm(128, 768, 3072)
    progs = [ls.ir.serialize(p) for p, _ in ls.spaces.sample_traces(e0, b200_space(pipeline=True), 96, seed=11)]
    res = plan(ls.ir.serialize(e0), progs)

    def unrolled(text):
        out = []

        def walk(stmts):
            for st in stmts:
                if "loop" in st:
                    if st["loop"]["kind"] == "unrolled":
                        out.append(st["loop"]["extent"])
                    walk(st["loop"]["body"])
        walk(json.loads(text)["root"])
        return out

    tc = [(p, r) for p, r in zip(progs, res) if r["family"] == "tcgen05"]
    assert len(tc) >= 8
    depths = set()
    for p, r in tc:
        u = unrolled(p)
        assert len(u) == 1
        if r["status"] == "OK":
            assert r["cfg"][6] == u[0], (r["cfg"], u)   # cfg[6] = stages
            depths.add(u[0])
        else:
            assert r["status"] == "ILLEGAL"
    assert len(depths) >= 3
    # fp32: the same traced depth in k-tiles is twice as many 32-element slots
    res32 = plan(ls.ir.serialize(e0), progs, dtype="f32")
    for p, r in zip(progs, res32):
        if r["family"] == "tcgen05" and r["status"] == "OK":
            assert r["cfg"][8] == 1 and r["cfg"][6] == 2 * unrolled(p)[0], (r["cfg"], unrolled(p))
