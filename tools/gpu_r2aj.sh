OUT=gpurun_out/r2aj; mkdir -p $OUT
L="variants/lib_is0.so variants/lib_is1.so"
timeout 900 python tools/k3_ab.py --libs $L --reps 14 > $OUT/ab_c3.txt 2>&1
timeout 600 python tools/k3_ab.py --libs $L --reps 14 --config c2 > $OUT/ab_c2.txt 2>&1
timeout 600 python tools/k3_ab.py --libs $L --reps 8 --config c4 > $OUT/ab_c4.txt 2>&1
timeout 600 python tools/k3_ab.py --libs $L --reps 3 --dense > $OUT/ab_dense.txt 2>&1
