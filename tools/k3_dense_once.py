"""One dense stage-3 launch (32 heads x 32K) after warm-up, for ncu captures."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2406_15486_b200 as sa
H, S = 32, int(sys.argv[1]) if len(sys.argv) > 1 else 32768
torch.manual_seed(0)
q, k, v = (torch.randn(n, S, 128, device="cuda", dtype=torch.bfloat16) for n in (H, 2, 2))
o = torch.empty_like(q)
for _ in range(3):
    sa.dense_attention(q, k, v, out=o)
torch.cuda.synchronize()
