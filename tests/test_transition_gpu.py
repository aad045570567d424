"""INT4 backup restore on the GPU vs the reference's own quantizer/dequantizer
(moeplan quant.py, imported unchanged): fp64 output bit-exact, bf16 output
equal to the reference value rounded fp64 -> fp32 -> bf16."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,group", [(1, 128), (7, 128), (1000, 128), (4097, 64), (100_003, 7), (1 << 20, 128)])
def test_int4_restore_bit_exact_vs_reference(n, group):
    from paper_2508_19373_b200.config import import_moeplan
    from paper_2508_19373_b200.transition import Int4Backup

    mp = import_moeplan()
    rng = np.random.default_rng(n)
    x = rng.standard_normal(n) * 0.02
    if n > 300:
        x[:group * 2] = 0.125  # constant groups: scale 0 path
    q = mp.quantize_int4(x, group)
    ref = mp.dequantize(q)
    bk = Int4Backup(q)
    out64 = torch.empty(n, dtype=torch.float64, device="cuda")
    bk.restore(out64)
    out16 = torch.empty(n + 8, dtype=torch.bfloat16, device="cuda")
    bk.restore(out16)
    torch.cuda.synchronize()
    assert np.array_equal(out64.cpu().numpy(), ref)  # bit-exact (no FMA contraction)
    want = torch.from_numpy(ref).to(torch.float32).to(torch.bfloat16)
    assert torch.equal(out16[:n].cpu(), want)
    # the paper's accuracy claim for per-group INT4: cosine > 0.99
    assert mp.quant.cosine_similarity(ref, x) > 0.99 if n > 1000 else True


def test_dequant_table_is_a_reference_table():
    from paper_2508_19373_b200.transition import dequant_table, measure_dequant_seconds

    meas = measure_dequant_seconds(range(10, 21))
    table = dequant_table(meas, max_log2=36)
    assert table.lookup(8, 3 << 20) >= table.lookup(8, 1 << 20) > 0
    assert table.lookup(1, 1 << 10) == meas[1 << 10]
