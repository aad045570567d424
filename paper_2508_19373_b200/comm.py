"""Collective plumbing for the HAP layout transitions (torch.distributed).

One process per GPU; NCCL over NVLink 5 / NVSwitch on the B200 box, gloo in
the CPU multi-process tests.  Groups are created from the ownership order in
``layout.RankLayout`` (every rank calls new_group for every group of a kind,
in the same order, as torch requires).  The collectives executed are exactly
the comm_volume rows (strategies.py:296-344): AllReduce for TP, AllGather /
ReduceScatter for the DP<->TP boundary, All-to-All for EP dispatch/combine.
"""

from __future__ import annotations

from typing import Dict, List, Optional, Tuple

import torch
import torch.distributed as dist

from .layout import RankLayout

GROUP_KINDS = ("attn_tp_group", "exp_tp_group", "gather_group", "a2a_group")


def _staged() -> bool:
    """gloo cannot run collectives on CUDA tensors: stage them through host
    memory.  Only the single-GPU validation of the multi-rank bench uses this
    (several ranks sharing one device, HAP_DIST_BACKEND=gloo); NCCL is the
    product backend."""
    return dist.is_initialized() and dist.get_backend() == "gloo"


class Comm:
    """Per-rank handles to the process groups a plan needs."""

    def __init__(self, lay: RankLayout):
        self.lay = lay
        self.staged = _staged()
        self.groups: Dict[str, Tuple[List[int], Optional[object]]] = {}
        distributed = dist.is_available() and dist.is_initialized()
        if lay.n > 1 and not distributed:
            raise RuntimeError("a plan over N > 1 devices needs torch.distributed to be initialised")
        if distributed and dist.get_world_size() != lay.n:
            raise RuntimeError(f"world size {dist.get_world_size()} != plan devices {lay.n}")
        for kind in GROUP_KINDS:
            mine = getattr(lay, kind)()
            handle = None
            for ranks in lay.all_groups(kind):
                if len(ranks) == 1:
                    continue
                g = dist.new_group(ranks=ranks) if len(ranks) < lay.n else dist.group.WORLD
                if lay.rank in ranks:
                    handle = g
            self.groups[kind] = (mine, handle)

    def size(self, kind: str) -> int:
        return len(self.groups[kind][0])

    def index(self, kind: str) -> int:
        return self.groups[kind][0].index(self.lay.rank)

    def _g(self, kind):
        return self.groups[kind][1]

    def enable_peer_allreduce(self, kinds, n_max: int = 1 << 20, mode: str = "peer") -> None:
        """Route all-reduces of bf16 tensors up to n_max elements on these groups
        through a one-shot kernel: "peer" = peer-memory reads (peer.PeerAllReduce),
        "nvls" = in-switch reduction over NVSwitch multicast memory
        (peer.NvlsAllReduce)."""
        from .peer import NvlsAllReduce, PeerAllReduce

        cls = NvlsAllReduce if mode == "nvls" else PeerAllReduce
        if not hasattr(self, "peer_ar"):
            self.peer_ar = {}
        for kind in kinds:
            if self.size(kind) > 1 and kind not in self.peer_ar:
                self.peer_ar[kind] = cls(n_max, torch.device("cuda", torch.cuda.current_device()), self._g(kind),
                                         self.groups[kind][0])

    def uses_peer_allreduce(self, kind: str) -> bool:
        return kind in getattr(self, "peer_ar", {})

    def barrier(self, kind: str) -> None:
        if self.size(kind) > 1:
            dist.barrier(group=self._g(kind))

    # All ops are no-ops on singleton groups.
    def all_reduce(self, t: torch.Tensor, kind: str) -> torch.Tensor:
        par = getattr(self, "peer_ar", {}).get(kind)
        if par is not None and par.fits(t):
            return par(t)
        if self.size(kind) > 1:
            if self.staged and t.is_cuda:
                h = t.cpu()
                dist.all_reduce(h, group=self._g(kind))
                t.copy_(h)
            else:
                dist.all_reduce(t, group=self._g(kind))
        return t

    def all_gather(self, out: torch.Tensor, inp: torch.Tensor, kind: str) -> torch.Tensor:
        if self.size(kind) == 1:
            if out.data_ptr() != inp.data_ptr():
                out.copy_(inp)
            return out
        if self.staged and out.is_cuda:
            h = torch.empty(out.shape, dtype=out.dtype)
            dist.all_gather_into_tensor(h, inp.contiguous().cpu(), group=self._g(kind))
            out.copy_(h)
            return out
        dist.all_gather_into_tensor(out, inp.contiguous(), group=self._g(kind))
        return out

    def reduce_scatter(self, out: torch.Tensor, inp: torch.Tensor, kind: str) -> torch.Tensor:
        if self.size(kind) == 1:
            if out.data_ptr() != inp.data_ptr():
                out.copy_(inp)
            return out
        if self.staged and out.is_cuda:
            h = torch.empty(out.shape, dtype=out.dtype)
            dist.reduce_scatter_tensor(h, inp.contiguous().cpu(), group=self._g(kind))
            out.copy_(h)
            return out
        dist.reduce_scatter_tensor(out, inp.contiguous(), group=self._g(kind))
        return out

    def all_to_all(self, out: torch.Tensor, inp: torch.Tensor, out_splits: List[int], in_splits: List[int],
                   kind: str) -> torch.Tensor:
        if self.size(kind) == 1:
            out.copy_(inp)
            return out
        if self.staged and out.is_cuda:
            h = torch.empty(out.shape, dtype=out.dtype)
            dist.all_to_all_single(h, inp.cpu(), output_split_sizes=out_splits, input_split_sizes=in_splits,
                                   group=self._g(kind))
            out.copy_(h)
            return out
        dist.all_to_all_single(out, inp, output_split_sizes=out_splits, input_split_sizes=in_splits,
                               group=self._g(kind))
        return out
