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


class PeerBoundary:
    """The DP<->TP boundary of one expert-TP group over peer memory
    (HAP_BOUNDARY_PEER=1): for plans whose gather group is the expert-TP group
    and attention is pure DP (e.g. the reference's roofline pick
    attn(dp=N) + exp(tp=N)).

    * all-gather: the RMSNorm that produces a replica's normalised rows stores
      them into that replica's row block of every rank's ``gath`` buffer
      (hap_rmsnorm_multi), then a device barrier;
    * reduce-scatter: the combine stores chunk q of its partial sums into slot
      ``me`` of rank q's ``slots`` buffer (hap_moe_combine_chunked), a device
      barrier, then each owner sums its slots in rank order
      (hap_reduce_slots_bf16).

    Both exchanges are stores issued by the kernels that produce the data (the
    NVLink transfer overlaps the norm / combine), and nothing synchronises the
    host, so a decode step under such a plan is CUDA-graph capturable.  One
    flag row per group serves every barrier (epochs only grow); single buffers
    are safe because each exchange is separated from the next write into the
    same buffer by the other exchange's barrier."""

    def __init__(self, rows: int, h: int, device, group, group_ranks: List[int]):
        self.rows, self.h = rows, h
        self.n = len(group_ranks)
        self.me = group_ranks.index(dist.get_rank())
        self.gath = PeerBuffer(self.n * rows, h, torch.bfloat16, device, group, group_ranks)
        self.slots = PeerBuffer(self.n * rows, h, torch.bfloat16, device, group, group_ranks)
        self.sig = PeerBuffer(1, self.n, torch.int32, device, group, group_ranks)
        self.sig.local.zero_()
        self.epoch = torch.zeros(1, dtype=torch.int32, device=device)
        torch.cuda.synchronize()
        dist.barrier(group=group)  # every flag row is zero before anyone publishes
        dev = self.epoch.device
        row_bytes = h * 2
        self.ag_tab = torch.tensor([p + self.me * rows * row_bytes for p in self.gath.ptrs], dtype=torch.int64,
                                   device=dev)
        self.rs_tab = torch.tensor(self.slots.ptrs, dtype=torch.int64, device=dev)
        self.sig_tab = torch.tensor(self.sig.ptrs, dtype=torch.int64, device=dev)

    def barrier(self) -> None:
        from . import ops

        ops.peer_barrier(self.sig_tab, self.epoch, self.n, self.me)

    def close(self) -> None:
        for b in (self.gath, self.slots, self.sig):
            b.close()


class PeerEP:
    """EP dispatch / combine over peer memory with the exchange planned on the
    device (HAP_EP_PEER=1): every rank pushes its permute segment offsets into
    every rank's ``segs`` table (hap_peer_broadcast_i32), a device barrier, then
    hap_ep_exchange_plan derives the receive offsets, the dispatch destinations
    and the combine targets on the device; hap_peer_copy_rows stores the rows
    into the owners' ``recv`` buffers, and the down GEMM's scatter epilogue
    stores the expert outputs back into the sources' ``y`` buffers.  Buffers are
    sized for the worst case (every row of every source routed here), so no
    count ever reaches the host: three device barriers per call and no host
    synchronisation (graph capturable)."""

    def __init__(self, rows: int, h: int, inter_local: int, n_experts: int, device, group,
                 group_ranks: List[int]):
        self.n = len(group_ranks)
        self.me = group_ranks.index(dist.get_rank())
        self.rows, self.E = rows, n_experts
        self.El = n_experts // self.n
        cap = self.n * rows
        self.segs = PeerBuffer(self.n, n_experts + 1, torch.int32, device, group, group_ranks)
        self.recv = PeerBuffer(cap, h, torch.bfloat16, device, group, group_ranks)
        self.y = PeerBuffer(rows, h, torch.bfloat16, device, group, group_ranks)
        self.sig = PeerBuffer(1, self.n, torch.int32, device, group, group_ranks)
        self.sig.local.zero_()
        self.epoch = torch.zeros(1, dtype=torch.int32, device=device)
        self.H = torch.empty(cap, inter_local, dtype=torch.bfloat16, device=device)
        torch.cuda.synchronize()
        dist.barrier(group=group)  # flags zero everywhere before anyone publishes
        dev = self.epoch.device
        i64 = dict(dtype=torch.int64, device=dev)
        self.segs_tab = torch.tensor(self.segs.ptrs, **i64)
        self.sig_tab = torch.tensor(self.sig.ptrs, **i64)
        self.dst_base = torch.tensor([self.recv.ptrs[e // self.El] for e in range(n_experts)], **i64)
        self.seg_dst = torch.tensor([self.y.ptrs[s] for s in range(self.n) for _ in range(self.El)], **i64)
        self.grp = torch.arange(self.El, dtype=torch.int32, device=dev).repeat(self.n)
        self.dst_row0 = torch.zeros(n_experts, **i64)
        self.seg_r = torch.zeros(n_experts + 1, dtype=torch.int32, device=dev)
        self.seg_dst_row0 = torch.zeros(n_experts, dtype=torch.int32, device=dev)

    def barrier(self) -> None:
        from . import ops

        ops.peer_barrier(self.sig_tab, self.epoch, self.n, self.me)

    def close(self) -> None:
        for b in (self.segs, self.recv, self.y, self.sig):
            b.close()


def _drv_check(res):
    """cuda.bindings.driver calls return (CUresult, *values)."""
    from cuda.bindings import driver as drv

    err, *vals = res if isinstance(res, tuple) else (res,)
    if err != drv.CUresult.CUDA_SUCCESS:
        raise RuntimeError(f"CUDA driver call failed: {err}")
    return vals[0] if len(vals) == 1 else (tuple(vals) if vals else None)


def nvls_supported(device: int, n_devices: int = 1) -> bool:
    """True when a multicast object can actually be created here: the device
    attribute alone is not enough — a B200 without an NVSwitch fabric reports
    CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED = 1 yet cuMulticastCreate fails
    with CUDA_ERROR_INVALID_VALUE (this run's one-GPU boxes)."""
    try:
        from cuda.bindings import driver as drv

        _drv_check(drv.cuInit(0))
        dev = _drv_check(drv.cuDeviceGet(device))
        attr = drv.CUdevice_attribute.CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED
        if not _drv_check(drv.cuDeviceGetAttribute(attr, dev)):
            return False
        prop = drv.CUmulticastObjectProp()
        prop.numDevices = n_devices
        prop.handleTypes = drv.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_FABRIC
        prop.flags = 0
        prop.size = 2 << 20
        prop.size = _drv_check(drv.cuMulticastGetGranularity(
            prop, drv.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_RECOMMENDED))
        handle = _drv_check(drv.cuMulticastCreate(prop))
        drv.cuMemRelease(handle)
        return True
    except Exception:  # noqa: BLE001 - no driver bindings / no multicast fabric: not supported
        return False


class NvlsAllReduce:
    """One-shot all-reduce through NVLink SHARP (HAP_NVLS_AR=1): one physical
    allocation per device bound to an NVSwitch multicast object
    (cuMulticastCreate / AddDevice / BindMem; the object travels between the
    ranks as a fabric handle), a unicast and a multicast mapping of it, and
    hap_nvls_allreduce_bf16 reducing in the switch (multimem.ld_reduce).  The
    caller (not the kernel library) owns every allocation, as the C ABI asks."""

    def __init__(self, n_max: int, device, group, group_ranks: List[int], n_ctas: int = 32):
        from cuda.bindings import driver as drv

        from . import _lib

        if n_max % 8:
            raise ValueError("n_max must be a multiple of 8")
        self.n_max, self.n_ctas = n_max, n_ctas
        self.n = len(group_ranks)
        self.me = group_ranks.index(dist.get_rank()) if dist.is_initialized() else 0
        dev_idx = torch.device(device).index if torch.device(device).index is not None else torch.cuda.current_device()
        _drv_check(drv.cuInit(0))
        cu_dev = _drv_check(drv.cuDeviceGet(dev_idx))
        need = int(_lib.load().hap_nvls_allreduce_bytes(n_max, n_ctas))
        fabric = drv.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_FABRIC
        mcprop = drv.CUmulticastObjectProp()
        mcprop.numDevices = self.n
        # the object crosses processes as a fabric handle; a one-device group
        # never exports it (a handle type is still required)
        mcprop.handleTypes = fabric if self.n > 1 else \
            drv.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR
        mcprop.flags = 0
        mcprop.size = need
        gran = _drv_check(drv.cuMulticastGetGranularity(
            mcprop, drv.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_RECOMMENDED))
        size = (need + gran - 1) // gran * gran
        mcprop.size = size
        # the multicast object: created by the group's first rank, imported by the others
        if self.me == 0:
            self.mc_handle = _drv_check(drv.cuMulticastCreate(mcprop))
            blob = bytes(_drv_check(drv.cuMemExportToShareableHandle(self.mc_handle, fabric, 0)).data) \
                if self.n > 1 else b""
        else:
            blob = None
        if self.n > 1:
            objs = [blob]
            dist.broadcast_object_list(objs, src=group_ranks[0], group=group)
            if self.me != 0:
                fh = drv.CUmemFabricHandle()
                fh.data = objs[0]
                self.mc_handle = _drv_check(drv.cuMemImportFromShareableHandle(fh, fabric))
        _drv_check(drv.cuMulticastAddDevice(self.mc_handle, cu_dev))
        if self.n > 1:
            dist.barrier(group=group)  # every device joined before memory is bound
        prop = drv.CUmemAllocationProp()
        prop.type = drv.CUmemAllocationType.CU_MEM_ALLOCATION_TYPE_PINNED
        prop.location.type = drv.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
        prop.location.id = dev_idx
        ugran = _drv_check(drv.cuMemGetAllocationGranularity(
            prop, drv.CUmemAllocationGranularity_flags.CU_MEM_ALLOC_GRANULARITY_RECOMMENDED))
        size = (size + ugran - 1) // ugran * ugran
        self.size = size
        self.mem = _drv_check(drv.cuMemCreate(size, prop, 0))
        _drv_check(drv.cuMulticastBindMem(self.mc_handle, 0, self.mem, 0, size, 0))
        access = drv.CUmemAccessDesc()
        access.location.type = drv.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
        access.location.id = dev_idx
        access.flags = drv.CUmemAccess_flags.CU_MEM_ACCESS_FLAGS_PROT_READWRITE
        self.uc = _drv_check(drv.cuMemAddressReserve(size, max(gran, ugran), 0, 0))
        _drv_check(drv.cuMemMap(self.uc, size, 0, self.mem, 0))
        _drv_check(drv.cuMemSetAccess(self.uc, size, [access], 1))
        self.mc = _drv_check(drv.cuMemAddressReserve(size, max(gran, ugran), 0, 0))
        _drv_check(drv.cuMemMap(self.mc, size, 0, self.mc_handle, 0))
        _drv_check(drv.cuMemSetAccess(self.mc, size, [access], 1))
        _drv_check(drv.cuMemsetD8(self.uc, 0, size))  # flag counters start at zero
        torch.cuda.synchronize()
        if self.n > 1:
            dist.barrier(group=group)
        self.epoch = torch.zeros(n_ctas, dtype=torch.int32, device=torch.device("cuda", dev_idx))

    def fits(self, t: torch.Tensor) -> bool:
        return t.dtype == torch.bfloat16 and t.is_contiguous() and t.numel() % 8 == 0 and t.numel() <= self.n_max

    def __call__(self, t: torch.Tensor, out: torch.Tensor = None) -> torch.Tensor:
        from . import ops

        out = t if out is None else out
        return ops.nvls_allreduce(t, out, int(self.uc), int(self.mc), self.epoch, self.n_max, self.n, self.n_ctas)

    def close(self) -> None:
        from cuda.bindings import driver as drv

        if getattr(self, "mem", None) is None:
            return
        torch.cuda.synchronize()
        for va in (self.uc, self.mc):
            drv.cuMemUnmap(va, self.size)
            drv.cuMemAddressFree(va, self.size)
        drv.cuMulticastUnbind(self.mc_handle, drv.cuDeviceGet(self.epoch.device.index)[1], 0, self.size)
        drv.cuMemRelease(self.mem)
        drv.cuMemRelease(self.mc_handle)
        self.mem = None
