# K1: S released after waiting for chunk 3 at chunk 2 (before the last 64 exponentials) vs after chunk 3's load (before the last 32)
OUT=gpurun_out/r2s3u; mkdir -p $OUT
L="variants/lib_k1r20.so variants/lib_k1r21.so"
timeout 600 python tools/exact_bench.py --libs $L --config c4 --chunk-n 77 --mode tensor --reps 5 > $OUT/k1r2_c4_77.txt 2>&1
timeout 600 python tools/exact_bench.py --libs variants/lib_k1r21.so variants/lib_k1r20.so --config c4 --chunk-n 77 --mode tensor --reps 5 >> $OUT/k1r2_c4_77.txt 2>&1
timeout 300 python tools/exact_bench.py --libs $L --config c3 --mode tensor --reps 10 > $OUT/k1r2_c3.txt 2>&1
timeout 300 python tools/exact_bench.py --libs $L --config c4 --mode tensor --reps 10 > $OUT/k1r2_c4_15.txt 2>&1
