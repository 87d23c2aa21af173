# fold / rowfin with batched loads (same summation order) vs the previous kernels: stage-1 A/B (tensor + exact), bit-identity
OUT=gpurun_out/r2s3i; mkdir -p $OUT
L="variants/lib_fold_old.so variants/lib_fold_new.so"
timeout 600 python tools/exact_bench.py --libs $L --config c4 --chunk-n 77 --mode tensor --reps 5 > $OUT/fold_c4_77.txt 2>&1
timeout 600 python tools/exact_bench.py --libs variants/lib_fold_new.so variants/lib_fold_old.so --config c4 --chunk-n 77 --mode tensor --reps 5 >> $OUT/fold_c4_77.txt 2>&1
timeout 300 python tools/exact_bench.py --libs $L --config c3 --mode tensor --reps 10 > $OUT/fold_c3.txt 2>&1
timeout 300 python tools/exact_bench.py --libs $L --config c2 --mode exact --reps 5 > $OUT/fold_c2_exact.txt 2>&1
