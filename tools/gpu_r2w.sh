OUT=gpurun_out/r2w; mkdir -p $OUT
L="variants/lib_f0.so variants/lib_f1.so variants/lib_f1e3.so variants/lib_f1e4.so"
timeout 900 python tools/k3_ab.py --libs $L --reps 12 > $OUT/ab_c3.txt 2>&1
timeout 600 python tools/k3_ab.py --libs $L --reps 4 --dense > $OUT/ab_dense.txt 2>&1
timeout 600 python tools/k3_ab.py --libs $L --reps 12 --config c2 > $OUT/ab_c2.txt 2>&1
