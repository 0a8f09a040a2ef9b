"""bench.py host-side arithmetic (no GPU): the algorithmic FLOPs and bytes
behind roofline.achieved / frac_attainable."""
import pytest

import bench


@pytest.mark.parametrize("workload,flops,nbytes", [
    # FLOPs = 2 M N K (x batch; conv 2 P Q K C R S); bytes = inputs once in the
    # runner dtype + the fp32 output once
    ("bert_ffn", 603_979_776, 128 * 3072 * 2 + 3072 * 768 * 2 + 128 * 768 * 4),
    ("bmm_qk", 25_165_824, 12 * 128 * 64 * 2 * 2 + 12 * 128 * 128 * 4),
    ("gmm512", 268_435_456, 3 * 512 * 512 * 4),
    ("conv2d", 231_211_008, 56 * 56 * 64 * 2 + 3 * 3 * 64 * 64 * 2 + 56 * 56 * 64 * 4),
])
def test_algorithmic_flops_and_bytes(workload, flops, nbytes):
    hdr, _ = bench.load_pop(workload)
    assert bench.contraction_flops(hdr["e0"]) == flops
    assert bench.algorithmic_bytes(hdr["e0"], bench.WORKLOADS[workload][1]) == nbytes


def test_every_bench_workload_has_a_population():
    for name, (pop, dtype, desc) in bench.WORKLOADS.items():
        hdr, progs = bench.load_pop(name)
        assert dtype in ("bf16", "f32") and desc and len(progs) >= 8 * 1024 or name == "conv2d_f32"
