OUT=gpurun_out/r2f; mkdir -p $OUT
L="variants/lib_e0.so variants/lib_e1.so variants/lib_e2.so variants/lib_e4.so"
timeout 600 python tools/k3_ab.py --libs $L --reps 12 > $OUT/ab_emu_c3.txt 2>&1
timeout 600 python tools/k3_ab.py --libs $L --reps 4 --dense > $OUT/ab_emu_dense.txt 2>&1
