# K1 releasing S as soon as the last TMEM load of pass 2 landed (before the last 32 exps) vs after the block's sums
OUT=gpurun_out/r2s3k; mkdir -p $OUT
L="variants/lib_k1er0.so variants/lib_k1er1.so"
timeout 600 python tools/exact_bench.py --libs $L --config c4 --chunk-n 77 --mode tensor --reps 5 > $OUT/k1er_c4_77.txt 2>&1
timeout 600 python tools/exact_bench.py --libs variants/lib_k1er1.so variants/lib_k1er0.so --config c4 --chunk-n 77 --mode tensor --reps 5 >> $OUT/k1er_c4_77.txt 2>&1
timeout 300 python tools/exact_bench.py --libs $L --config c3 --mode tensor --reps 10 > $OUT/k1er_c3.txt 2>&1
timeout 300 python tools/exact_bench.py --libs $L --config c4 --mode tensor --reps 10 > $OUT/k1er_c4_15.txt 2>&1
