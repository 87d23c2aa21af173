OUT=gpurun_out/r2as; mkdir -p $OUT
L="variants/lib_sc0.so variants/lib_sc1.so"
timeout 300 python tools/k3_ab.py --libs $L --reps 14 > $OUT/ab_c3.txt 2>&1
timeout 200 python tools/k3_ab.py --libs $L --reps 14 --config c2 > $OUT/ab_c2.txt 2>&1
timeout 300 python tools/k3_ab.py --libs $L --reps 3 --dense > $OUT/ab_dense.txt 2>&1
