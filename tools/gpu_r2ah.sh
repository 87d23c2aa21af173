OUT=gpurun_out/r2ah; mkdir -p $OUT
L="variants/lib_xold.so variants/lib_xnew.so"
timeout 600 python tools/exact_bench.py --libs $L --config c2 --reps 6 > $OUT/exact_c2.txt 2>&1
timeout 600 python tools/exact_bench.py --libs $L --config c3 --reps 4 > $OUT/exact_c3.txt 2>&1
timeout 600 python tools/exact_bench.py --libs $L --config c4 --chunk-n 31 --reps 3 > $OUT/exact_c4_31.txt 2>&1
