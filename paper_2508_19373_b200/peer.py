"""Peer-mapped device buffers for the EP dispatch / combine over NVLink.

``PeerBuffer`` allocates one device buffer per rank of a process group and maps
every peer's buffer into this process through CUDA IPC (the handles travel
over the group with ``all_gather_object``; opening them enables peer access,
so kernel stores to a peer address go over NVLink / NVSwitch).  The executor's
EP path uses two of them: the expert-side receive buffer (dispatch rows are
copied straight into it by ``hap_peer_copy_rows``) and the token-side expert
output buffer (the down-projection GEMM's scatter epilogue writes each expert
output straight back to its source rank) — the two all-to-alls of
strategies.py:334-338 done as direct stores from the kernels that produce the
data.  The same mechanism maps buffers of several ranks sharing one GPU (the
single-GPU validation mode of the multi-rank tests).
"""

from __future__ import annotations

from typing import List

import torch
import torch.distributed as dist


class PeerBuffer:
    def __init__(self, rows: int, cols: int, dtype, device, group, group_ranks: List[int]):
        from torch.multiprocessing.reductions import reduce_tensor

        self.rows, self.cols = rows, cols
        self.local = torch.empty(rows, cols, dtype=dtype, device=device)
        fn, args = reduce_tensor(self.local)
        objs = [None] * len(group_ranks)
        dist.all_gather_object(objs, (dist.get_rank(), fn, args), group=group)
        me = dist.get_rank()
        self.views = []
        for r, f, a in objs:
            self.views.append(self.local if r == me else f(*a))
        from . import _lib

        lib = _lib.load()
        for v in self.views:  # stores from this device go straight over NVLink
            if v.device != self.local.device:
                _lib.check(lib.hap_enable_peer_access(v.device.index), "hap_enable_peer_access")
        self.ptrs = [v.data_ptr() for v in self.views]  # group order

    def __len__(self):
        return len(self.views)

    def close(self) -> None:
        """Drop the peer mappings (call on every rank before a barrier, ahead of shutdown)."""
        self.views = [self.local]
        self.ptrs = []
