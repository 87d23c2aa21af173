OUT=gpurun_out/r2ax; mkdir -p $OUT
timeout 600 python tools/guard_kinds.py 32768 1 2 ref > $OUT/kinds_c2ref.txt 2>&1
timeout 300 python tools/guard_kinds.py 131072 1 2 > $OUT/kinds_c3.txt 2>&1
