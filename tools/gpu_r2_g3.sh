OUT=gpurun_out/r2g3; mkdir -p $OUT
timeout 600 python tools/band_w_diag.py 32768 2 ref > $OUT/band_w_c2ref.txt 2>&1
timeout 600 python tools/band_w_diag.py 32768 2 > $OUT/band_w_c2.txt 2>&1
