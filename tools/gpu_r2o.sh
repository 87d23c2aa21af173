OUT=gpurun_out/r2o; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden_metrics.py tests/test_tuning.py -m gpu -q > $OUT/pytest_parity.log 2>&1
timeout 600 python bench.py --no-cpu --no-dense > $OUT/bench_c3.json 2> $OUT/bench_c3.err
