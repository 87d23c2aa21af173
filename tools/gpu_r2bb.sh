OUT=gpurun_out/r2bb; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.log 2>&1
timeout 300 python bench.py --no-cpu --no-dense --no-e2e > $OUT/bench_c3.json 2> $OUT/bench.err
timeout 300 python bench.py --config c4 --chunk-n 77 --no-cpu --no-dense --no-e2e > $OUT/bench_c4_r10.json 2>> $OUT/bench.err
timeout 300 python bench.py --config c4 --no-cpu --no-dense --no-e2e > $OUT/bench_c4.json 2>> $OUT/bench.err
timeout 300 python tools/rownorm_diag.py 98304 77 8 > $OUT/rn_c4_77.txt 2>&1
timeout 300 python tools/rownorm_diag.py 131072 1 2 > $OUT/rn_c3.txt 2>&1
timeout 300 python tools/guard_diag.py 98304 77 > $OUT/guard_c4_77.txt 2>&1
