"""hap_copy2d_batched (the reshard's pack / unpack copy engine): many strided
row-stack copies in one launch are byte-identical to torch's copy_, across
row sizes that straddle the 16 KB chunk, single-row and many-row records, more
records than one launch carries, and argument errors rejected before launch."""

import pytest
import torch

from paper_2508_19373_b200 import _lib, ops

pytestmark = pytest.mark.gpu


def _rand(shape, dtype=torch.bfloat16):
    return torch.randint(-30000, 30000, shape, device="cuda", dtype=torch.int16).view(dtype)


@pytest.mark.parametrize("n_pairs", [1, 7, 500])
def test_batched_copy_matches_torch(n_pairs):
    g = torch.Generator().manual_seed(n_pairs)
    pairs, want = [], []
    for i in range(n_pairs):
        rows = int(torch.randint(1, 40, (1,), generator=g))
        cols = 8 * int(torch.randint(1, 2600, (1,), generator=g))  # up to ~41 KB rows: 1-3 chunks
        src_full = _rand((rows, cols + 8 * int(torch.randint(0, 4, (1,), generator=g))))
        src = src_full[:, :cols]
        dst_full = _rand((rows, cols + 16))
        dst = dst_full[:, 8:8 + cols]
        ref = dst_full.clone()
        ref[:, 8:8 + cols] = src
        pairs.append((src, dst))
        want.append((dst_full, ref))
    moved = ops.copy_views(pairs)
    torch.cuda.synchronize()
    assert moved == sum(s.numel() * 2 for s, _ in pairs)
    for got, ref in want:
        assert torch.equal(got.view(torch.int16), ref.view(torch.int16))  # padding columns untouched too


def test_batched_copy_interleaved_blocks():
    # the reshard's gate rows: [n/hw, hw, h] blocks of an interleaved [2I, h] tensor
    I, h, hw = 1792, 1024, 128
    w13 = _rand((2 * I, h))
    v = w13.view(I // hw, 2, hw, h)
    gate = torch.empty(I // hw, hw, h, device="cuda", dtype=torch.bfloat16)
    up = torch.empty_like(gate)
    ops.copy_views([(v[:, 0], gate), (v[:, 1], up)])
    torch.cuda.synchronize()
    bits = lambda t: t.contiguous().view(torch.int16)  # noqa: E731  (random bit patterns include NaNs)
    assert torch.equal(bits(gate), bits(v[:, 0])) and torch.equal(bits(up), bits(v[:, 1]))


def test_batched_copy_rejects_bad_records():
    import numpy as np

    lib = _lib.load()
    a = torch.empty(4096, device="cuda", dtype=torch.uint8)
    rec = np.array([[a.data_ptr() + 8, a.data_ptr() + 2048, 1, 64, 64, 64]], dtype=np.int64)
    assert lib.hap_copy2d_batched(rec.ctypes.data, 1, 0) == -3  # misaligned source
    rec = np.array([[a.data_ptr(), a.data_ptr() + 2048, 2, 64, 32, 64]], dtype=np.int64)
    assert lib.hap_copy2d_batched(rec.ctypes.data, 1, 0) == -1  # pitch shorter than the row
    with pytest.raises(ValueError):
        ops.copy_views([(a[:64].view(8, 8).t(), a[64:128].view(8, 8))])  # column-major view: not a row stack
