OUT=gpurun_out/r2h; mkdir -p $OUT
L="variants/lib_e0.so variants/lib_e1.so variants/lib_l0.so variants/lib_l1.so"
timeout 900 python tools/k3_ab.py --libs $L --reps 16 > $OUT/ab_c3.txt 2>&1
timeout 600 python tools/k3_ab.py --libs $L --reps 16 --config c2 > $OUT/ab_c2.txt 2>&1
timeout 600 python tools/k3_ab.py --libs $L --reps 8 --config c4 > $OUT/ab_c4.txt 2>&1
timeout 600 python tools/k3_ab.py --libs $L --reps 4 --dense > $OUT/ab_dense.txt 2>&1
