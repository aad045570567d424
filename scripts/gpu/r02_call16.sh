for o in 0 1 0 1; do HAP_ATTN_OPT=$o timeout 120 python scripts/attn_opt_ab.py; done
python -c "
import torch; a=torch.load('/tmp/attn_opt_0.pt'); b=torch.load('/tmp/attn_opt_1.pt'); print('bit-identical:', torch.equal(a,b), (a.float()-b.float()).abs().max().item())"
timeout 300 python -m pytest tests/test_kernels_gpu.py -m gpu -q -x -k "attn" 2>&1 | tail -2
