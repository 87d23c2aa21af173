OUT=gpurun_out/r2y; mkdir -p $OUT
timeout 600 python tools/exact_bench.py --libs variants/lib_xlib.so variants/lib_xnew.so --config c2 --reps 6 > $OUT/exact_c2.txt 2>&1
timeout 600 python tools/exact_bench.py --libs variants/lib_xlib.so variants/lib_xnew.so --config c3 --reps 4 > $OUT/exact_c3.txt 2>&1
