"""TEST DOUBLE: torch-CPU implementations of the executor's op interface.

Used only by the gloo multi-process tests (tests/test_executor_dist.py) to
exercise the HAP collective schedule and layout transitions on CPU, where
the sm_100a kernels cannot run.  The product executor never imports this
(its default ``CudaOps`` calls libhap_kernels.so exclusively).  Semantics
mirror include/hap_kernels.h: fp32 math, one bf16 rounding per stored tensor.
"""

from __future__ import annotations

import torch

BF16 = torch.bfloat16


def _swiglu_cols(acc: torch.Tensor, hw: int) -> torch.Tensor:
    M, N = acc.shape
    a = acc.view(M, N // (2 * hw), 2, hw)
    g, u = a[:, :, 0], a[:, :, 1]
    return (g / (1 + torch.exp(-g)) * u).reshape(M, N // 2)


class CpuOps:
    @staticmethod
    def rmsnorm(x, w, eps, out=None):
        xf = x.float()
        y = xf * torch.rsqrt((xf * xf).mean(-1, keepdim=True) + eps) * w.float()
        if out is None:
            return y.to(BF16)
        out.copy_(y)
        return out

    @staticmethod
    def gemm(a, w, out=None, *, bias=None, residual=None, swiglu_half=0, sm_budget=0):
        acc = a.float() @ w.float().t()
        if swiglu_half:
            acc = _swiglu_cols(acc, swiglu_half)
        if bias is not None:
            acc = acc + bias.float()
        if residual is not None:
            acc = acc + residual.float()
        if out is None:
            return acc.to(BF16)
        out.copy_(acc)
        return out

    @staticmethod
    def gemm_qkv_rope(a, w, pos, n_rope_heads, d, theta, bias=None, out=None):
        qkv = CpuOps.gemm(a, w, bias=bias)
        T = qkv.shape[0]
        inv = 1.0 / (theta ** (torch.arange(0, d, 2, dtype=torch.float64) / d))
        ang = pos.double()[:, None] * inv[None, :]
        cos, sin = torch.cos(ang).float()[:, None, :], torch.sin(ang).float()[:, None, :]
        acc = a.float() @ w.float().t()
        if bias is not None:
            acc = acc + bias.float()
        x = acc[:, :n_rope_heads * d].view(T, n_rope_heads, d)
        x1, x2 = x[..., :d // 2], x[..., d // 2:]
        y = torch.cat([x1 * cos - x2 * sin, x2 * cos + x1 * sin], -1)
        qkv[:, :n_rope_heads * d] = y.reshape(T, -1).to(BF16)
        return qkv

    @staticmethod
    def grouped_gemm(a, b, n_groups, seg, out, *, swiglu_half=0, bias=None, residual=None, seg_group=None):
        b3 = b.reshape(n_groups, -1, b.shape[-1])
        segs = seg.tolist()
        groups = seg_group.tolist() if seg_group is not None else list(range(len(segs) - 1))
        for s in range(len(segs) - 1):
            r0, r1 = segs[s], segs[s + 1]
            if r1 > r0:
                acc = a[r0:r1].float() @ b3[groups[s]].float().t()
                if swiglu_half:
                    acc = _swiglu_cols(acc, swiglu_half)
                out[r0:r1] = acc.to(BF16)
        return out

    @staticmethod
    def rope_qk(qkv, nq, nkv, d, pos, theta):
        T = qkv.shape[0]
        inv = 1.0 / (theta ** (torch.arange(0, d, 2, dtype=torch.float64) / d))
        ang = pos.double()[:, None] * inv[None, :]
        cos, sin = torch.cos(ang).float()[:, None, :], torch.sin(ang).float()[:, None, :]
        x = qkv[:, :(nq + nkv) * d].float().view(T, nq + nkv, d)
        x1, x2 = x[..., :d // 2], x[..., d // 2:]
        y = torch.cat([x1 * cos - x2 * sin, x2 * cos + x1 * sin], -1)
        qkv[:, :(nq + nkv) * d] = y.reshape(T, -1).to(BF16)

    @staticmethod
    def _attend(q, k, v, causal_offset=None):
        # q [S, Hq, d], k/v [L, Hkv, d]
        S, Hq, d = q.shape
        L, Hkv, _ = k.shape
        rep = Hq // Hkv
        kk = k.float().repeat_interleave(rep, 1)
        vv = v.float().repeat_interleave(rep, 1)
        s = torch.einsum("shd,lhd->hsl", q.float(), kk) / d ** 0.5
        qpos = torch.arange(L - S, L)[:, None]
        mask = torch.arange(L)[None, :] <= qpos
        s = s.masked_fill(~mask[None], float("-inf"))
        p = torch.softmax(s, -1)
        return torch.einsum("hsl,lhd->shd", p, vv)

    @staticmethod
    def attn_prefill(qkv, nq, nkv, d, n_seqs, S, out, causal=True):
        for s in range(n_seqs):
            blk = qkv[s * S:(s + 1) * S]
            q = blk[:, :nq * d].view(S, nq, d)
            k = blk[:, nq * d:(nq + nkv) * d].view(S, nkv, d)
            v = blk[:, (nq + nkv) * d:(nq + 2 * nkv) * d].view(S, nkv, d)
            out[s * S:(s + 1) * S] = CpuOps._attend(q, k, v).reshape(S, -1).to(BF16)
        return out

    @staticmethod
    def kv_cache_fill(qkv, nq, nkv, d, n_seqs, S, kc, vc):
        for s in range(n_seqs):
            blk = qkv[s * S:(s + 1) * S]
            kc[s, :, :S] = blk[:, nq * d:(nq + nkv) * d].view(S, nkv, d).transpose(0, 1)
            vc[s, :, :S] = blk[:, (nq + nkv) * d:(nq + 2 * nkv) * d].view(S, nkv, d).transpose(0, 1)

    @staticmethod
    def attn_decode(qkv, kc, vc, pos, nq, nkv, d, out, ws):
        B = qkv.shape[0]
        for b in range(B):
            p = int(pos[b])
            kc[b, :, p] = qkv[b, nq * d:(nq + nkv) * d].view(nkv, d)
            vc[b, :, p] = qkv[b, (nq + nkv) * d:(nq + 2 * nkv) * d].view(nkv, d)
            q = qkv[b, :nq * d].view(1, nq, d)
            k = kc[b, :, :p + 1].transpose(0, 1)
            v = vc[b, :, :p + 1].transpose(0, 1)
            out[b] = CpuOps._attend(q, k, v).reshape(-1).to(BF16)
        return out

    @staticmethod
    def router_topk(x, w, E, k, renorm, has_shared, idx, tw, sg=None, logits=None):
        lg = x.float() @ w.float().t()
        order = torch.sort(-lg[:, :E], dim=-1, stable=True).indices[:, :k]
        p = torch.softmax(lg[:, :E].double(), -1)
        sel = torch.gather(p, 1, order)
        if renorm:
            sel = sel / sel.sum(-1, keepdim=True)
        idx.copy_(order.to(torch.int32))
        tw.copy_(sel.float())
        if has_shared and sg is not None:
            sg.copy_(torch.sigmoid(lg[:, E]))

    @staticmethod
    def moe_permute(eid, E, x, div, x_out, dst, seg, ws):
        e = eid.long()
        valid = (e >= 0) & (e < E)
        counts = torch.bincount(e[valid], minlength=E)
        seg[0] = 0
        seg[1:] = torch.cumsum(counts, 0).to(torch.int32)
        rows = torch.nonzero(valid).view(-1)
        order = rows[torch.sort(e[rows], stable=True).indices]
        d = torch.full_like(e, -1)
        d[order] = torch.arange(order.numel())
        dst.copy_(d.to(torch.int32))
        if x_out is not None and order.numel():
            x_out[:order.numel()] = x[order // div]

    @staticmethod
    def moe_combine(y, dst, tw, T, k, out, residual=None, shared_y=None, shared_gate=None, res_row0=0,
                    res_rows=None):
        d = dst.view(T, k).long()
        acc = torch.zeros(T, out.shape[1])
        for j in range(k):
            ok = d[:, j] >= 0
            acc[ok] += tw.view(T, k)[ok, j, None] * y[d[ok, j]].float()
        if shared_y is not None:
            acc += shared_gate[:, None] * shared_y.float()
        if residual is not None:
            n = residual.shape[0] if res_rows is None else res_rows
            acc[res_row0:res_row0 + n] += residual[:n].float()
        out.copy_(acc)

    @staticmethod
    def permute_workspace_bytes(rows, E):
        return 16

    @staticmethod
    def attn_decode_workspace_bytes(B, nq, d, max_len):
        return 16
