OUT=gpurun_out/r2g; mkdir -p $OUT
L="variants/lib_e0.so variants/lib_e1.so variants/lib_e5.so variants/lib_e6.so variants/lib_e7.so variants/lib_e8.so"
timeout 900 python tools/k3_ab.py --libs $L --reps 16 > $OUT/ab_emu_c3.txt 2>&1
timeout 600 python tools/k3_ab.py --libs $L --reps 16 --config c2 > $OUT/ab_emu_c2.txt 2>&1
