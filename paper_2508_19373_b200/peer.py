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


class PeerAllReduce:
    """One-shot all-reduce over a process group through peer-mapped memory
    (hap_peer_allreduce_bf16): symmetric data (2 x n_max bf16) and flag regions,
    a local epoch per CTA, and device tables of addresses.  The per-call input
    address is written into the table by a fill kernel, so the call is
    CUDA-graph capturable (no host synchronisation, no NCCL)."""

    def __init__(self, n_max: int, device, group, group_ranks: List[int], n_ctas: int = 32):
        from . import _lib

        if n_max % 8:
            raise ValueError("n_max must be a multiple of 8")
        self.n_max, self.n_ctas = n_max, n_ctas
        self.n = len(group_ranks)
        self.me = group_ranks.index(dist.get_rank())
        sig_elems = int(_lib.load().hap_peer_allreduce_sig_bytes(self.n, n_ctas)) // 4
        self.data = PeerBuffer(2, n_max, torch.bfloat16, device, group, group_ranks)
        self.sig = PeerBuffer(1, sig_elems, torch.int32, device, group, group_ranks)
        self.sig.local.zero_()
        self.epoch = torch.zeros(n_ctas, dtype=torch.int32, device=device)
        torch.cuda.synchronize()
        dist.barrier(group=group)  # every rank's flags are zero before anyone publishes
        dev = self.epoch.device
        self.data_tab = torch.tensor(self.data.ptrs, dtype=torch.int64, device=dev)
        self.sig_tab = torch.tensor(self.sig.ptrs, dtype=torch.int64, device=dev)
        self.epoch_tab = torch.zeros(self.n, dtype=torch.int64, device=dev)
        self.epoch_tab[self.me] = self.epoch.data_ptr()
        self.io_tab = torch.zeros(self.n, dtype=torch.int64, device=dev)

    def fits(self, t: torch.Tensor) -> bool:
        return t.dtype == torch.bfloat16 and t.is_contiguous() and t.numel() % 8 == 0 and t.numel() <= self.n_max

    def __call__(self, t: torch.Tensor) -> torch.Tensor:
        from . import ops

        self.io_tab[self.me].fill_(t.data_ptr())
        ops.peer_allreduce(self.io_tab, self.io_tab, self.epoch_tab, self.data_tab, self.sig_tab, t.numel(),
                           self.n_max, self.n, self.me, 1, self.n_ctas)
        return t

    def close(self) -> None:
        self.data.close()
        self.sig.close()
