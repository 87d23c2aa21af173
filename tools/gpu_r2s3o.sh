# K1 with the K tile as two 64-dim halves (each half of K(j+1) loads when QK^T(j) is done with it) vs whole-tile ring
OUT=gpurun_out/r2s3o; mkdir -p $OUT
L="variants/lib_k1hk0.so variants/lib_k1hk1.so"
timeout 600 python tools/exact_bench.py --libs $L --config c4 --chunk-n 77 --mode tensor --reps 5 > $OUT/k1hk_c4_77.txt 2>&1
timeout 600 python tools/exact_bench.py --libs variants/lib_k1hk1.so variants/lib_k1hk0.so --config c4 --chunk-n 77 --mode tensor --reps 5 >> $OUT/k1hk_c4_77.txt 2>&1
timeout 300 python tools/exact_bench.py --libs $L --config c3 --mode tensor --reps 10 > $OUT/k1hk_c3.txt 2>&1
timeout 300 python tools/exact_bench.py --libs $L --config c4 --mode tensor --reps 10 > $OUT/k1hk_c4_15.txt 2>&1
