OUT=gpurun_out/r2ap; mkdir -p $OUT
L="variants/lib_k1e0.so variants/lib_k1e1.so"
timeout 300 python tools/exact_bench.py --libs $L --config c3 --mode tensor --reps 10 > $OUT/k1_c3.txt 2>&1
timeout 300 python tools/exact_bench.py --libs $L --config c4 --chunk-n 77 --mode tensor --reps 5 > $OUT/k1_c4_77.txt 2>&1
SA_LIB_PATH=variants/lib_k1e1.so timeout 300 python tools/guard_diag.py 131072 1 > $OUT/guard_c3.txt 2>&1
SA_LIB_PATH=variants/lib_k1e1.so timeout 300 python tools/guard_diag.py 98304 77 > $OUT/guard_c4_77.txt 2>&1
