OUT=gpurun_out/r2af; mkdir -p $OUT
L="variants/lib_sw0.so variants/lib_sw1.so variants/lib_sw2.so"
timeout 900 python tools/k3_ab.py --libs $L --reps 12 > $OUT/ab_c3.txt 2>&1
timeout 600 python tools/k3_ab.py --libs $L --reps 3 --dense > $OUT/ab_dense.txt 2>&1
