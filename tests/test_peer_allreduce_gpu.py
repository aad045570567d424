"""One-shot peer all-reduce kernel, all ranks played by one launch on one B200
(their CTAs co-resident, so the flag barrier is exercised for real): the sum
is bit-identical on every rank and equals the rank-ordered fp32 sum rounded
once to bf16; repeated calls (epochs, parity buffers) and CUDA-graph replay."""

import pytest
import torch

pytestmark = pytest.mark.gpu


def _setup(n_ranks, n_max, n_ctas):
    from paper_2508_19373_b200 import _lib

    sig_bytes = _lib.load().hap_peer_allreduce_sig_bytes(n_ranks, n_ctas)
    data = [torch.zeros(2 * n_max, device="cuda", dtype=torch.bfloat16) for _ in range(n_ranks)]
    sig = [torch.zeros(sig_bytes // 4, device="cuda", dtype=torch.int32) for _ in range(n_ranks)]
    epoch = [torch.zeros(n_ctas, device="cuda", dtype=torch.int32) for _ in range(n_ranks)]
    tab = lambda ts: torch.tensor([t.data_ptr() for t in ts], device="cuda", dtype=torch.int64)  # noqa: E731
    return data, sig, epoch, tab


@pytest.mark.parametrize("n_ranks", [2, 4, 8])
def test_peer_allreduce_simulated_ranks(n_ranks):
    from paper_2508_19373_b200 import ops

    n_max, n_ctas = 64 * 4096, 32
    data, sig, epoch, tab = _setup(n_ranks, n_max, n_ctas)
    for call, n in enumerate([64 * 4096, 8 * 4096, 64 * 4096, 1024]):
        ins = [torch.randn(n, device="cuda").to(torch.bfloat16) for _ in range(n_ranks)]
        outs = [torch.empty_like(x) for x in ins]
        ops.peer_allreduce(tab(ins), tab(outs), tab(epoch), tab(data), tab(sig), n, n_max, n_ranks, 0, n_ranks,
                           n_ctas)
        torch.cuda.synchronize()
        ref = torch.zeros(n, device="cuda")
        for x in ins:
            ref += x.float()
        ref = ref.to(torch.bfloat16)
        for o in outs:
            assert torch.equal(o, ref), f"call {call}"
        assert all(int(e.min()) == call + 1 and int(e.max()) == call + 1 for e in epoch)


def test_peer_allreduce_in_place_graph_replay():
    from paper_2508_19373_b200 import ops

    n_ranks, n_max, n_ctas, n = 4, 32 * 4096, 16, 32 * 4096
    data, sig, epoch, tab = _setup(n_ranks, n_max, n_ctas)
    bufs = [torch.empty(n, device="cuda", dtype=torch.bfloat16) for _ in range(n_ranks)]
    tables = [tab(bufs), tab(epoch), tab(data), tab(sig)]

    def step():
        ops.peer_allreduce(tables[0], tables[0], tables[1], tables[2], tables[3], n, n_max, n_ranks, 0, n_ranks,
                           n_ctas)

    src = [torch.randn(n, device="cuda").to(torch.bfloat16) for _ in range(n_ranks)]
    for b, s in zip(bufs, src):
        b.copy_(s)
    step()  # warm-up outside capture
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        step()
    for rep in range(3):
        src = [torch.randn(n, device="cuda").to(torch.bfloat16) for _ in range(n_ranks)]
        for b, s in zip(bufs, src):
            b.copy_(s)
        g.replay()
        torch.cuda.synchronize()
        ref = torch.zeros(n, device="cuda")
        for s in src:
            ref += s.float()
        ref = ref.to(torch.bfloat16)
        assert all(torch.equal(b, ref) for b in bufs), rep


def test_tp_decode_peer_allreduce_two_ranks(tmp_path):
    """Pure-TP decode on two ranks sharing the GPU: the block's all-reduces go
    through the peer kernel (HAP_PEER_AR=1), match the gloo path within bf16
    tolerance, and the step is graph-captured (no NCCL, no host sync) and
    replays to the same bytes.  (Two contexts time-slice the GPU, so the flag
    barrier is slow here but exercised across processes.)"""
    import json
    import socket
    import subprocess
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parents[1]
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    out = str(tmp_path / "res")
    procs = [subprocess.Popen([sys.executable, str(root / "tests" / "peer_ar_worker.py"),
                               json.dumps(dict(rank=r, world=2, port=port, out=out))]) for r in range(2)]
    try:
        for p in procs:
            assert p.wait(timeout=240) == 0
    finally:
        for p in procs:
            if p.poll() is None:
                p.kill()
    res = [torch.load(f"{out}.{r}") for r in range(2)]
    assert all(r["ok"] for r in res), res
