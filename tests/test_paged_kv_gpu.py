"""Paged KV cache (the full-model loop with KV bytes that
grow per decode step, reference simulate.py:78-114, arch.py:193-201).

The paged entry points run the same arithmetic as the contiguous ones (same
split plan for the same max_len, same 16-key chunks), so outputs must be
bit-identical:
  * kernel level: a contiguous cache copied into shuffled pages, one decode
    step (append + attention) on both;
  * model level: two stacked blocks, prefill then decode steps that cross page
    boundaries (pages handed out as the sequences grow), eager and from a CUDA
    graph whose block-table rows are refreshed in place between replays.
"""

import pytest
import torch

pytestmark = pytest.mark.gpu
dev = torch.device("cuda")


def test_paged_decode_kernel_matches_contiguous():
    from paper_2508_19373_b200 import ops

    B, nq, nkv, d, max_len, page = 3, 8, 2, 128, 512, 64
    g = torch.Generator(device=dev).manual_seed(3)
    kc = torch.randn(B, nkv, max_len, d, device=dev, generator=g).to(torch.bfloat16)
    vc = torch.randn(B, nkv, max_len, d, device=dev, generator=g).to(torch.bfloat16)
    qkv = torch.randn(B, (nq + 2 * nkv) * d, device=dev, generator=g).to(torch.bfloat16)
    pos = torch.tensor([37, 150, 511], device=dev, dtype=torch.int32)
    mp = max_len // page
    n_pages = B * mp + 5
    perm = torch.randperm(n_pages, generator=torch.Generator().manual_seed(1))[:B * mp].view(B, mp).to(torch.int32)
    kp = torch.zeros(n_pages, nkv, page, d, device=dev, dtype=torch.bfloat16)
    vp = torch.zeros_like(kp)
    for b in range(B):
        for j in range(mp):
            kp[perm[b, j]] = kc[b, :, j * page:(j + 1) * page]
            vp[perm[b, j]] = vc[b, :, j * page:(j + 1) * page]
    table = perm.to(dev).contiguous()
    ws = torch.empty(ops.attn_decode_workspace_bytes(B, nq, d, max_len), device=dev, dtype=torch.uint8)
    out_c = torch.empty(B, nq * d, device=dev, dtype=torch.bfloat16)
    out_p = torch.empty_like(out_c)
    ops.attn_decode(qkv, kc, vc, pos, nq, nkv, d, out_c, ws)
    ops.attn_decode_paged(qkv, kp, vp, table, pos, nq, nkv, d, out_p, ws)
    torch.cuda.synchronize()
    assert torch.equal(out_c, out_p)
    for b in range(B):  # the appended row landed in the page holding position pos[b]
        p = int(pos[b])
        pg = int(perm[b, p // page])
        assert torch.equal(kp[pg, :, p % page], kc[b, :, p]) and torch.equal(vp[pg, :, p % page], vc[b, :, p])


@pytest.mark.parametrize("graph", [False, True], ids=["eager", "graph"])
def test_paged_model_loop_matches_contiguous(graph):
    from paper_2508_19373_b200.config import get_config
    from paper_2508_19373_b200.layout import PlanDegrees
    from paper_2508_19373_b200.model import HapModel

    cfg = get_config("tiny")
    L, B, S, steps, max_len, page = 2, 3, 100, 40, 160, 32
    model = HapModel(cfg, PlanDegrees(1, 1, 1, 1), None, n_layers=L, seed=5)
    g = torch.Generator(device=dev).manual_seed(7)
    x = torch.randn(B * S, cfg.hidden, device=dev, generator=g).to(torch.bfloat16)
    xs = [torch.randn(B, cfg.hidden, device=dev, generator=g).to(torch.bfloat16) for _ in range(steps)]
    runs = {}
    for paged in (False, True):
        caches = model.new_caches(B, max_len, paged=paged, page=page)
        outs = [model.prefill(x, B, S, caches)]
        pos = torch.full((B,), S, device=dev, dtype=torch.int32)
        if graph:
            xd = xs[0].clone()
            if paged:
                caches[0].state.ensure(S + 1)
            gr, gout = model.capture_decode(xd, B, caches, pos)
        for step in range(steps):
            if graph:
                if paged:  # the next token's page, table refreshed in place before the replay
                    caches[0].state.ensure(S + step + 1)
                xd.copy_(xs[step])
                gr.replay()
                outs.append(gout.clone())
                pos += 1
            else:
                outs.append(model.decode_step(xs[step], B, caches, pos, max_position=S + step))
                pos += 1
        torch.cuda.synchronize()
        runs[paged] = outs
        if paged:
            st = caches[0].state
            assert sum(st.held) == B * -(-(S + steps) // page)  # pages grew with the sequences
    for a, b in zip(runs[False], runs[True]):
        assert torch.equal(a, b)
