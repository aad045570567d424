"""Prefill->decode expert layout switch with the weights on the GPU: 2 and 4
ranks sharing one B200 (gloo-staged all-to-all; NCCL over NVLink on a multi-GPU
box) reshard between every pair of the catalog's expert strategies and must
reproduce the destination layout's packed weights exactly (SURVEY §8(f) row 1,
reference transition.py:127-177)."""

import json
import socket
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]
CFG = dict(name="mixtral-rs-test", n_layers=1, n_q_heads=8, n_kv_heads=2, head_dim=128, hidden=1024, n_experts=8,
           n_shared=0, top_k=2, inter=1792)
QCFG = dict(name="qwen-rs-test", n_layers=1, n_q_heads=8, n_kv_heads=8, head_dim=128, hidden=1024, n_experts=8,
            n_shared=2, top_k=4, inter=512, norm_topk_prob=False, qkv_bias=True, rms_eps=1e-6)


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("cfg,world", [(CFG, 2), (CFG, 4), (QCFG, 2)], ids=["mixtral-n2", "mixtral-n4", "qwen-n2"])
def test_reshard_on_gpu_matches_direct_pack(tmp_path, cfg, world):
    strat = [(t, world // t) for t in (1, 2, 4, 8) if t <= world and world % t == 0]
    pairs = [(a, b) for a in strat for b in strat if a != b]
    port = free_port()
    out = str(tmp_path / "res")
    procs = [subprocess.Popen([sys.executable, str(ROOT / "tests" / "reshard_gpu_worker.py"),
                               json.dumps(dict(rank=r, world=world, port=port, cfg=cfg, pairs=pairs, out=out))])
             for r in range(world)]
    for p in procs:
        assert p.wait(timeout=600) == 0
    for r in range(world):
        res = json.loads(Path(f"{out}.{r}").read_text())
        assert len(res) == len(pairs)
        assert all(v["ok"] for v in res.values()), res
