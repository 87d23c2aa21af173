"""Cycle accounting of the stage-3 kernel (library built with -DSA_K3_PROF=1):
per processed block, average cycles each role spends in each phase."""
import ctypes, os, sys, signal
signal.signal(signal.SIGPIPE, signal.SIG_DFL)
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2406_15486_b200 as sa
from paper_2406_15486_b200 import _lib
H, S = 32, int(sys.argv[1]) if len(sys.argv) > 1 else 32768
torch.manual_seed(0)
q, k, v = (torch.randn(n, S, 128, device="cuda", dtype=torch.bfloat16) for n in (H, 2, 2))
o = torch.empty_like(q)
lib = _lib.load()
buf = (ctypes.c_ulonglong * 16)()
sa.dense_attention(q, k, v, out=o); torch.cuda.synchronize()
lib.sa_debug_k3_profile(buf, 1)
sa.dense_attention(q, k, v, out=o); torch.cuda.synchronize()
lib.sa_debug_k3_profile(buf, 1)
v_ = list(buf)
blocks = v_[12]
names = ["sm: wait S", "sm: pass1 max", "sm: rescale", "sm: pass2 exp", "sm: wait O (epi)",
         "mma: wait P part", "mma: wait V", "mma: wait P full", "mma: wait K", "tma: wait K slot", "tma: wait V slot"]
print("blocks", blocks, "avg CTA cycles per block", v_[11] / max(1, blocks))
for i, nm in enumerate(names):
    div = blocks * (4 if i < 5 else 1)
    print(f"{nm:20s} {v_[i] / max(1, div):10.1f} cycles/block")
