OUT=gpurun_out/r2am; mkdir -p $OUT
timeout 300 python tools/guard_kinds.py 131072 1 2 > $OUT/kinds_c3.txt 2>&1
timeout 600 python tools/guard_kinds.py 98304 77 8 > $OUT/kinds_c4_77.txt 2>&1
timeout 300 python tools/guard_kinds.py 98304 15 8 > $OUT/kinds_c4_15.txt 2>&1
