import sys, torch
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2406_15486_b200 as sa
from paper_2406_15486_b200 import synth
S, Hq, Hkv = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
q, k, v, _ = synth.make_inputs(S, Hq, Hkv, 128, seed=1, device="cuda")
o, r = sa.sample_attention(q, k, v, alpha=0.95, chunk_n=1)
torch.cuda.synchronize()
print("ok", S, Hq, Hkv, float(o.float().abs().max()))
