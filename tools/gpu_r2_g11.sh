OUT=gpurun_out/r2g11; mkdir -p $OUT
nvidia-smi --query-gpu=clocks.sm,power.draw --format=csv > $OUT/gpu.txt
timeout 900 python tools/k3_ab.py --libs tools/ablibs/lib_prod.so tools/ablibs/lib_emu0.so tools/ablibs/lib_emu16.so --reps 60 > $OUT/k3_emu_power_ab.txt 2>&1
timeout 900 python tools/k3_ab.py --libs tools/ablibs/lib_emu0.so tools/ablibs/lib_prod.so tools/ablibs/lib_emu16.so --reps 60 >> $OUT/k3_emu_power_ab.txt 2>&1
