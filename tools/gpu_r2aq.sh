OUT=gpurun_out/r2aq; mkdir -p $OUT
L="variants/lib_k1c2.so variants/lib_k1c3.so"
timeout 120 python tools/exact_bench.py --libs $L --config c3 --mode tensor --reps 10 > $OUT/k1_c3.txt 2>&1
timeout 120 python tools/exact_bench.py --libs $L --config c4 --mode tensor --reps 10 > $OUT/k1_c4_15.txt 2>&1
timeout 200 python tools/exact_bench.py --libs $L --config c4 --chunk-n 77 --mode tensor --reps 5 > $OUT/k1_c4_77.txt 2>&1
