OUT=gpurun_out/r2at; mkdir -p $OUT
L="variants/lib_rf0.so variants/lib_rf1.so"
timeout 200 python tools/exact_bench.py --libs $L --config c4 --chunk-n 77 --mode tensor --reps 6 > $OUT/s1_c4_77.txt 2>&1
timeout 120 python tools/exact_bench.py --libs $L --config c3 --mode tensor --reps 10 > $OUT/s1_c3.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.log 2>&1
