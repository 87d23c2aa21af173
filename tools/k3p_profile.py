"""Cycle accounting of the paired stage-3 kernel (-DSA_K3_PROF=1)."""
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
lib.sa_debug_k3p_profile(buf, 1)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); sa.dense_attention(q, k, v, out=o); e1.record(); torch.cuda.synchronize()
lib.sa_debug_k3p_profile(buf, 1)
v_ = list(buf)
blocks = v_[12]
print("ms", e0.elapsed_time(e1), "blocks", blocks)
names = {0: ("sm: wait S", 4), 1: ("sm: pass1", 4), 2: ("sm: pass2+", 4), 3: ("mma: wait P part", 1),
         4: ("mma: wait V", 1), 5: ("mma: wait P full", 1), 6: ("mma: wait K", 1)}
for i, (nm, w) in names.items():
    print(f"{nm:20s} {v_[i] / max(1, blocks * w):10.1f} cycles/block")
