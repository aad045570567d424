"""Host-side page management of the paged KV cache (CPU): pages are handed out
as sequences grow, shared by every layer through one block table, returned on
release, and over-long sequences / an exhausted pool are rejected."""

import pytest
import torch

from paper_2508_19373_b200.executor import PagedKV, PagedKVCache


def test_pages_follow_sequence_growth_and_release():
    st = PagedKV(n_layers=3, batch=2, n_kv_local=2, head_dim=64, max_len=100, device="cpu", page=32)
    assert st.max_pages == 4 and st.max_len == 128 and st.n_pages == 8
    st.ensure(1)
    assert st.held == [1, 1] and (st.table[:, 0] >= 0).all() and (st.table[:, 1:] == -1).all()
    st.ensure(33, seqs=[1])
    assert st.held == [1, 2]
    ids = st.table_host[st.table_host >= 0].tolist()
    assert len(ids) == len(set(ids)) == 3          # no page handed out twice
    layers = [st.layer(i) for i in range(3)]
    assert all(isinstance(c, PagedKVCache) and c.state is st for c in layers)
    assert layers[0].k.shape == (8, 2, 32, 64) and layers[2].v.data_ptr() != layers[0].v.data_ptr()
    st.release(1)
    assert st.held == [1, 0] and (st.table[1] == -1).all() and len(st.free) == 7
    with pytest.raises(ValueError):
        st.ensure(129)
    with pytest.raises(ValueError, match="multiple of 16"):
        PagedKV(1, 1, 1, 64, 64, "cpu", page=24)


def test_pool_exhaustion_raises():
    st = PagedKV(n_layers=1, batch=2, n_kv_local=1, head_dim=64, max_len=64, device="cpu", page=16, n_pages=5)
    with pytest.raises(RuntimeError, match="out of pages"):
        st.ensure(48)


def test_positions_checked_against_paged_capacity():
    st = PagedKV(n_layers=1, batch=2, n_kv_local=1, head_dim=64, max_len=64, device="cpu", page=16)
    c = st.layer(0)
    assert c.check_positions(torch.tensor([3, 63], dtype=torch.int32)) == 63
    with pytest.raises(ValueError, match="outside the KV cache"):
        c.check_positions(torch.tensor([3, 64], dtype=torch.int32))
