"""Rank layout for one (AttentionStrategy, ExpertStrategy) plan.

Device ranks follow the reference's ownership order (transition.py:127-150,
``_ownership``): for the expert module rank = dp * (tp*ep) + ep_group * tp +
tp_rank; EP group g owns the contiguous expert block [g*E/ep, (g+1)*E/ep);
TP rank r owns the contiguous intermediate slice [r*I/tp, (r+1)*I/tp) of
every held expert; shared units are replicated across EP and DP and sliced
per unit by TP.  Attention uses the same convention: rank = dp_idx * tp +
tp_rank, heads [r*H/tp, (r+1)*H/tp).

Token layouts
-------------
Attention replica d (ranks [d*a_tp, (d+1)*a_tp)) owns the sequences
[d*ceil(B/a_dp), ...) (the planner's ceil split, planner.py:229), held
replicated on its a_tp ranks.  The expert module partitions tokens into
S_e = N / e_tp shards (shard = rank // e_tp), each replicated on its e_tp
consecutive ranks.  With that numbering every rank's expert shard either
lies inside its own attention replica (S_e >= a_dp: a local slice, no
communication) or is a union of whole replicas (S_e < a_dp: all-gather over
``gather_group``) — the DP->TP "boundary" of comm_volume (strategies.py:324-332).
"""

from __future__ import annotations

from dataclasses import dataclass
from math import ceil
from typing import List, Tuple


def _pow2(x: int) -> bool:
    return x >= 1 and (x & (x - 1)) == 0


@dataclass(frozen=True)
class PlanDegrees:
    """Plain degrees of a plan; built from moeplan strategies or by hand."""

    a_tp: int
    a_dp: int
    e_tp: int
    e_ep: int
    e_dp: int = 1

    @classmethod
    def from_strategies(cls, attention, expert) -> "PlanDegrees":
        return cls(a_tp=attention.tp_degree, a_dp=attention.dp_degree, e_tp=expert.tp_degree,
                   e_ep=expert.ep_degree, e_dp=getattr(expert, "dp_degree", 1))

    @property
    def n(self) -> int:
        return self.a_tp * self.a_dp

    def label(self) -> str:
        e = f"exp(tp={self.e_tp},ep={self.e_ep}" + (f",dp={self.e_dp})" if self.e_dp > 1 else ")")
        return f"attn(tp={self.a_tp},dp={self.a_dp})+{e}"


@dataclass(frozen=True)
class RankLayout:
    deg: PlanDegrees
    rank: int
    n_q_heads: int
    n_kv_heads: int
    n_experts: int
    inter: int
    n_shared: int

    def __post_init__(self):
        d = self.deg
        n = d.n
        if d.e_tp * d.e_ep * d.e_dp != n:
            raise ValueError(f"{d.label()}: strategies cover different device counts")
        if not (_pow2(d.a_tp) and _pow2(d.e_tp)):
            raise ValueError("TP degrees must be powers of two (strategies.py:75,100)")
        if self.n_q_heads % d.a_tp or self.n_kv_heads % d.a_tp:
            raise ValueError("attention tp must divide q and kv heads (strategies.py:77-80)")
        if self.n_experts % d.e_ep:
            raise ValueError("ep must divide n_experts (strategies.py:102-103)")
        if self.inter % d.e_tp:
            raise ValueError("expert tp must divide expert_inter_dim (strategies.py:104-107)")
        if d.e_dp > 1 and d.e_ep > 1:
            raise ValueError("DP and EP may not be combined (strategies.py:108-109)")
        if not 0 <= self.rank < n:
            raise ValueError(f"rank {self.rank} outside [0, {n})")

    # ------------------------------------------------------------ attention --
    @property
    def n(self) -> int:
        return self.deg.n

    @property
    def a_rep(self) -> int:
        return self.rank // self.deg.a_tp

    @property
    def a_tp_rank(self) -> int:
        return self.rank % self.deg.a_tp

    @property
    def q_heads(self) -> Tuple[int, int]:
        per = self.n_q_heads // self.deg.a_tp
        return self.a_tp_rank * per, (self.a_tp_rank + 1) * per

    @property
    def kv_heads(self) -> Tuple[int, int]:
        per = self.n_kv_heads // self.deg.a_tp
        return self.a_tp_rank * per, (self.a_tp_rank + 1) * per

    # --------------------------------------------------------------- expert --
    @property
    def e_rep(self) -> int:
        return self.rank // (self.deg.e_tp * self.deg.e_ep)

    @property
    def ep_group(self) -> int:
        return (self.rank % (self.deg.e_tp * self.deg.e_ep)) // self.deg.e_tp

    @property
    def e_tp_rank(self) -> int:
        return self.rank % self.deg.e_tp

    @property
    def experts(self) -> Tuple[int, int]:
        per = self.n_experts // self.deg.e_ep
        return self.ep_group * per, (self.ep_group + 1) * per

    @property
    def inter_slice(self) -> Tuple[int, int]:
        span = self.inter // self.deg.e_tp
        return self.e_tp_rank * span, (self.e_tp_rank + 1) * span

    def shared_rows(self) -> List[Tuple[int, int]]:
        """Row ranges of the wide shared MLP held here: per unit u the TP slice
        [u*I + r*I/tp, u*I + (r+1)*I/tp) (transition.py:147-149)."""
        i0, i1 = self.inter_slice
        return [(u * self.inter + i0, u * self.inter + i1) for u in range(self.n_shared)]

    @property
    def shard(self) -> int:
        return self.rank // self.deg.e_tp

    @property
    def n_shards(self) -> int:
        return self.n // self.deg.e_tp

    # --------------------------------------------------------------- groups --
    def attn_tp_group(self) -> List[int]:
        return [self.a_rep * self.deg.a_tp + j for j in range(self.deg.a_tp)]

    def exp_tp_group(self) -> List[int]:
        return [self.shard * self.deg.e_tp + j for j in range(self.deg.e_tp)]

    def gather_group(self) -> List[int]:
        """Ranks whose attention replicas make up this rank's expert shard
        (one per replica, same attention tp rank); size a_dp / S_e."""
        if self.n_shards >= self.deg.a_dp:
            return [self.rank]
        return [r for r in self.exp_tp_group() if r % self.deg.a_tp == self.a_tp_rank]

    def a2a_group(self) -> List[int]:
        """EP dispatch/combine group: same replica, same tp rank, every EP group."""
        d = self.deg
        base = self.e_rep * d.e_tp * d.e_ep
        return [base + g * d.e_tp + self.e_tp_rank for g in range(d.e_ep)]

    def all_groups(self, kind: str) -> List[List[int]]:
        """Every group of `kind` over all ranks (identical on every rank, for new_group)."""
        seen, out = set(), []
        for r in range(self.n):
            other = RankLayout(self.deg, r, self.n_q_heads, self.n_kv_heads, self.n_experts, self.inter,
                               self.n_shared)
            g = tuple(getattr(other, kind)())
            if g not in seen:
                seen.add(g)
                out.append(list(g))
        return out


def tokens_per_replica(batch: int, a_dp: int, seq: int, n: int) -> Tuple[int, int]:
    """(sequences per attention replica, padded token rows per replica).

    Rows are padded to a multiple of n so every all-gather / reduce-scatter
    chunking of a replica or shard divides evenly.
    """
    bpr = ceil(batch / a_dp)
    rows = bpr * seq
    rows = ceil(rows / n) * n
    return bpr, rows


def replica_sequences(batch: int, a_dp: int, rep: int) -> Tuple[int, int]:
    bpr = ceil(batch / a_dp)
    s0 = min(batch, rep * bpr)
    return s0, min(batch, s0 + bpr)
