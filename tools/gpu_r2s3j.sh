# fold / rowfin load batch: 4/4 vs 8/8 vs 16/8
OUT=gpurun_out/r2s3j; mkdir -p $OUT
L="variants/lib_fold_f4r4.so variants/lib_fold_f8r8.so variants/lib_fold_f16r8.so"
timeout 600 python tools/exact_bench.py --libs $L --config c4 --chunk-n 77 --mode tensor --reps 5 > $OUT/foldb_c4_77.txt 2>&1
timeout 300 python tools/exact_bench.py --libs $L --config c3 --mode tensor --reps 10 > $OUT/foldb_c3.txt 2>&1
timeout 300 python tools/exact_bench.py --libs $L --config c2 --mode exact --reps 5 > $OUT/foldb_c2_exact.txt 2>&1
