OUT=gpurun_out/r2an; mkdir -p $OUT
timeout 300 python tools/rownorm_diag.py 131072 1 2 > $OUT/rn_c3.txt 2>&1
timeout 600 python tools/rownorm_diag.py 98304 77 8 > $OUT/rn_c4_77.txt 2>&1
timeout 300 python tools/rownorm_diag.py 32768 1 2 > $OUT/rn_c2.txt 2>&1
