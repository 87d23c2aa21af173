OUT=gpurun_out/r2e; mkdir -p $OUT
timeout 1500 python tools/k3_ab.py --libs variants/lib_e0.so variants/lib_e1.so variants/lib_e2.so variants/lib_e3.so variants/lib_e4.so --rounds 3 --reps 4 > $OUT/ab_emu.txt 2>&1
