"""Per-kernel SASS summary of libsampleattn.so (cuobjdump -sass, sm_100a):
instruction count and the opcodes that show tcgen05 / TMA / TMEM / DMMA /
packed fp32 math.  Also writes the full SASS of the named hot kernels.

    python tools/sass_summary.py out_summary.txt out_hot.txt
"""
import collections
import re
import subprocess
import sys

LIB = "paper_2406_15486_b200/libsampleattn.so"
KEYS = ["UTCHMMA", "UTCBAR", "UTMALDG", "UTMAPF", "LDTM", "STTM", "MUFU.EX2", "FFMA2", "FADD2", "FMUL2", "FMNMX3",
        "DMMA", "DFMA", "SYNCS", "BAR.SYNC", "SHFL", "ELECT"]
HOT = ("k3_share", "k1_tc", "xf_itemsI13", "k_band_scores")

sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
funcs = collections.OrderedDict()
cur = None
for line in sass.splitlines():
    m = re.match(r"\s+Function : (\S+)", line)
    if m:
        cur = m.group(1)
        funcs[cur] = []
        continue
    if cur and re.match(r"\s+/\*[0-9a-f]{4,}\*/", line):
        funcs[cur].append(line)
out = ["# SASS summary of libsampleattn.so (cuobjdump -sass, sm_100a), round 2",
       "# per kernel: instruction count and the opcodes proving tcgen05 / TMA / TMEM / DMMA / packed math", ""]
for name, lines in funcs.items():
    counts = collections.Counter()
    for ln in lines:
        op = re.sub(r"^\s+/\*[0-9a-f]+\*/\s+(@!?U?P\w+\s+)?", "", ln).split()[0] if ln.strip() else ""
        for k in KEYS:
            if op.startswith(k):
                counts[k] += 1
    out.append(name)
    out.append(f"  instructions={len(lines)} " + " ".join(f"{k}={counts[k]}" for k in KEYS if counts[k]))
open(sys.argv[1], "w").write("\n".join(out) + "\n")
with open(sys.argv[2], "w") as f:
    for name, lines in funcs.items():
        if any(h in name for h in HOT):
            f.write(f"\n\n===== {name}\n")
            f.write("\n".join(lines))
print(len(funcs), "kernels")
