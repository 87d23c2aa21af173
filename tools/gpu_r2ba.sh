OUT=gpurun_out/r2ba; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.log 2>&1
timeout 300 python bench.py --no-cpu --no-dense --no-e2e > $OUT/bench_c3.json 2> $OUT/bench.err
timeout 300 python bench.py --config c4 --chunk-n 77 --no-cpu --no-dense --no-e2e > $OUT/bench_c4_r10.json 2>> $OUT/bench.err
