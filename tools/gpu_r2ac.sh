OUT=gpurun_out/r2ac; mkdir -p $OUT
L="variants/lib_k1old.so variants/lib_k1new.so"
timeout 600 python tools/exact_bench.py --libs $L --config c3 --mode tensor --reps 10 > $OUT/k1_c3.txt 2>&1
timeout 600 python tools/exact_bench.py --libs $L --config c4 --chunk-n 77 --mode tensor --reps 5 > $OUT/k1_c4_77.txt 2>&1
timeout 600 python tools/exact_bench.py --libs $L --config c4 --mode tensor --reps 10 > $OUT/k1_c4_15.txt 2>&1
