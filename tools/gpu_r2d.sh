OUT=gpurun_out/r2d; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_golden_metrics.py tests/test_gpu_parity.py -m gpu -q -rA > $OUT/pytest_gpu.log 2>&1
timeout 900 python bench.py --no-e2e > $OUT/bench_c3.json 2> $OUT/bench_c3.err
