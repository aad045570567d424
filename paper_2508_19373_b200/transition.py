"""Stage-switch machinery of HAP's Eq.6 (reference
transition.py:1-267): the INT4 quantized-backup path measured on B200.

* ``Int4Backup`` keeps a GQI4 tensor (the reference's own container,
  quant.py:19-22, 119-154) in pinned host memory and restores it on device:
  asynchronous H2D upload of codes/scales/zero points, then the
  ``hap_int4_dequant`` kernel (bit-exact vs quant.py:dequantize in fp64, or
  bf16 weights).
* ``measure_dequant_table`` / ``measure_h2d_bandwidth`` produce the planner's
  inputs from measurements: a reference ``DequantTimeTable`` (transition.py:
  46-124; CSV ``n_gpus,v_dequant,seconds``) and ``host_to_device_bw`` for
  ``HardwareProfile`` (arch.py:80-101), replacing the synthetic 20e9
  params/s table (transition.py:36, 84-97).
"""

from __future__ import annotations

import statistics
from typing import Dict, Tuple

import torch

from . import ops as K
from .config import import_moeplan


class Int4Backup:
    """A GQI4 tensor resident in pinned host memory."""

    def __init__(self, q):
        self.group_size = int(q.group_size)
        self.n = int(q.original_len)
        self.codes = torch.from_numpy(q.codes.copy()).pin_memory()
        self.scales = torch.from_numpy(q.scales.copy()).pin_memory()
        self.zeros = torch.from_numpy(q.zero_points.copy()).pin_memory()

    @classmethod
    def from_values(cls, values, group_size: int = 128) -> "Int4Backup":
        mp = import_moeplan()
        return cls(mp.quantize_int4(values, group_size))

    def nbytes(self) -> int:
        return self.codes.numel() + 8 * (self.scales.numel() + self.zeros.numel())

    def restore(self, out: torch.Tensor, stream: torch.cuda.Stream = None) -> torch.Tensor:
        """Upload + dequantize into ``out`` (float64 or bf16, >= n elements) on ``stream``."""
        dev = out.device
        stream = stream or torch.cuda.current_stream(dev)
        with torch.cuda.stream(stream):
            codes = torch.empty(((self.codes.numel() + 3) // 4) * 4, dtype=torch.uint8, device=dev)
            codes[:self.codes.numel()].copy_(self.codes, non_blocking=True)
            scales = self.scales.to(dev, non_blocking=True)
            zeros = self.zeros.to(dev, non_blocking=True)
            K.int4_dequant(codes, scales, zeros, self.group_size, self.n, out)
        return out


def _time(fn, reps: int = 5) -> float:
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        s = torch.cuda.Event(enable_timing=True)
        e = torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e) / 1e3)
    return statistics.median(ts)


def measure_dequant_seconds(log2_sizes=range(10, 32), group_size: int = 128) -> Dict[int, float]:
    """Device seconds to dequantize 2^k parameters into bf16 (one B200)."""
    out: Dict[int, float] = {}
    max_n = 1 << max(log2_sizes)
    codes = torch.randint(0, 256, ((max_n + 1) // 2,), dtype=torch.uint8, device="cuda")
    n_groups = (max_n + group_size - 1) // group_size
    scales = torch.rand(n_groups, dtype=torch.float64, device="cuda") * 1e-2
    zeros = torch.randn(n_groups, dtype=torch.float64, device="cuda") * 1e-2
    dst = torch.empty(max_n, dtype=torch.bfloat16, device="cuda")
    for lg in log2_sizes:
        n = 1 << lg
        out[n] = _time(lambda: K.int4_dequant(codes, scales, zeros, group_size, n, dst))
    del codes, scales, zeros, dst
    torch.cuda.empty_cache()
    return out


def dequant_table(measured: Dict[int, float], max_gpus: int = 16, max_log2: int = 40):
    """Reference DequantTimeTable from per-device measurements.  Each device
    dequantizes its own shard concurrently, so every n_gpus row is the
    single-device curve; buckets beyond the largest measured size are
    extrapolated at the measured asymptotic rate (largest bucket)."""
    mp = import_moeplan()
    sizes = sorted(measured)
    top = sizes[-1]
    rate = top / measured[top]
    entries: Dict[Tuple[int, int], float] = {}
    n = 1
    while n <= max_gpus:
        for lg in range(10, max_log2 + 1):
            b = 1 << lg
            entries[(n, b)] = measured[b] if b in measured else max(measured[top], b / rate)
        n *= 2
    # enforce monotone rows (the reference table contract)
    for n2 in {k[0] for k in entries}:
        prev = 0.0
        for lg in range(10, max_log2 + 1):
            key = (n2, 1 << lg)
            entries[key] = max(entries[key], prev)
            prev = entries[key]
    return mp.DequantTimeTable(entries=entries)


def measure_h2d_bandwidth(nbytes: int = 1 << 30, reps: int = 5) -> float:
    """Pinned host -> device copy bandwidth (bytes/s)."""
    src = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    dst = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    t = _time(lambda: dst.copy_(src, non_blocking=True), reps)
    return nbytes / t
