OUT=gpurun_out/r2g12; mkdir -p $OUT
timeout 900 python tools/k3_ab.py --libs tools/ablibs/lib_prod.so tools/ablibs/lib_emu316.so tools/ablibs/lib_emu14.so --reps 60 > $OUT/k3_emu_power_ab2.txt 2>&1
timeout 900 python tools/k3_ab.py --libs tools/ablibs/lib_emu14.so tools/ablibs/lib_emu316.so tools/ablibs/lib_prod.so --reps 60 >> $OUT/k3_emu_power_ab2.txt 2>&1
