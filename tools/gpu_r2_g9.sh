OUT=gpurun_out/r2g9; mkdir -p $OUT
timeout 900 python tools/guard_kinds.py 131072 1 2 ref > $OUT/guard_kinds_c3ref.txt 2>&1
timeout 900 python tools/band_w_diag.py 131072 2 ref > $OUT/band_w_c3ref.txt 2>&1
