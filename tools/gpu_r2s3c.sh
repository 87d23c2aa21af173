# K1 with two q heads per CTA (shared K tile) vs one head per CTA: interleaved stage-1 A/B, bit-identity, parity tests
OUT=gpurun_out/r2s3c; mkdir -p $OUT
L="variants/lib_k1p0.so variants/lib_k1p1.so"
timeout 300 python tools/exact_bench.py --libs $L --config c3 --mode tensor --reps 10 > $OUT/k1pair_c3.txt 2>&1
timeout 300 python tools/exact_bench.py --libs $L --config c2 --mode tensor --reps 10 > $OUT/k1pair_c2.txt 2>&1
timeout 300 python tools/exact_bench.py --libs $L --config c4 --mode tensor --reps 10 > $OUT/k1pair_c4_15.txt 2>&1
timeout 600 python tools/exact_bench.py --libs $L --config c4 --chunk-n 77 --mode tensor --reps 5 > $OUT/k1pair_c4_77.txt 2>&1
timeout 600 python tools/exact_bench.py --libs variants/lib_k1p1.so variants/lib_k1p0.so --config c4 --chunk-n 77 --mode tensor --reps 5 >> $OUT/k1pair_c4_77.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -x > $OUT/pytest_parity.txt 2>&1
