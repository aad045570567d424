"""NVLS (NVLink SHARP) one-shot all-reduce: the multicast object, its unicast
and multicast mappings, and the multimem.red / multimem.ld_reduce kernel.
On a box with an NVSwitch fabric, a one-device group's in-switch sum must
return the input bit for bit, across repeated epochs (counter and
parity-buffer protocol), in place, and from a CUDA graph.  This run's one-GPU
boxes report multicast support but cannot create multicast objects
(cuMulticastCreate -> CUDA_ERROR_INVALID_VALUE, scripts/diag/mc_create.py), so
the tests skip there; the kernel compiles to LDGMC / multimem REDG."""

import pytest
import torch

pytestmark = pytest.mark.gpu


def _nvls():
    from paper_2508_19373_b200.peer import NvlsAllReduce, nvls_supported

    if not nvls_supported(0):
        pytest.skip("no NVSwitch multicast fabric on this box (cuMulticastCreate unavailable)")
    return NvlsAllReduce(1 << 16, torch.device("cuda", 0), None, [0], n_ctas=16)


def test_nvls_allreduce_single_device_identity():
    ar = _nvls()
    g = torch.Generator(device="cuda").manual_seed(3)
    try:
        for n in (8, 4096, 65536, 24576):
            x = torch.randn(n, device="cuda", generator=g).to(torch.bfloat16)
            out = torch.empty_like(x)
            ar(x, out)
            torch.cuda.synchronize()
            assert torch.equal(out, x), n
        y = torch.randn(4096, device="cuda", generator=g).to(torch.bfloat16)
        y0 = y.clone()
        ar(y)  # in place
        torch.cuda.synchronize()
        assert torch.equal(y, y0)
        assert int(ar.epoch.min()) == int(ar.epoch.max()) == 5
    finally:
        ar.close()


def test_nvls_allreduce_graph_replay():
    ar = _nvls()
    try:
        x = torch.randn(8192, device="cuda").to(torch.bfloat16)
        out = torch.empty_like(x)
        ar(x, out)
        torch.cuda.synchronize()
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr):
            ar(x, out)
        for _ in range(3):
            out.zero_()
            gr.replay()
            torch.cuda.synchronize()
            assert torch.equal(out, x)
    finally:
        ar.close()
