# K1: pass 2's first TMEM load issued at the end of pass 1 vs at the start of pass 2
OUT=gpurun_out/r2s3m; mkdir -p $OUT
L="variants/lib_k1pf0.so variants/lib_k1pf1.so"
timeout 600 python tools/exact_bench.py --libs $L --config c4 --chunk-n 77 --mode tensor --reps 5 > $OUT/k1pf_c4_77.txt 2>&1
timeout 600 python tools/exact_bench.py --libs variants/lib_k1pf1.so variants/lib_k1pf0.so --config c4 --chunk-n 77 --mode tensor --reps 5 >> $OUT/k1pf_c4_77.txt 2>&1
timeout 300 python tools/exact_bench.py --libs $L --config c3 --mode tensor --reps 10 > $OUT/k1pf_c3.txt 2>&1
timeout 300 python tools/exact_bench.py --libs $L --config c4 --mode tensor --reps 10 > $OUT/k1pf_c4_15.txt 2>&1
