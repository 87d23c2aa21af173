OUT=gpurun_out/r2c; mkdir -p $OUT
timeout 300 python tools/guard_diag.py 131072 1 > $OUT/guard_c3.txt 2>&1
timeout 300 python tools/guard_diag.py 98304 77 > $OUT/guard_c4_77.txt 2>&1
timeout 300 python tools/guard_large_logits.py > $OUT/guard_large.txt 2>&1
timeout 900 python bench.py --no-cpu --no-e2e > $OUT/bench_c3.json 2> $OUT/bench_c3.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
