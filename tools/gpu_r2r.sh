OUT=gpurun_out/r2r; mkdir -p $OUT
timeout 600 python tools/e2e_diag.py > $OUT/e2e_diag.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden_metrics.py -m gpu -q -x > $OUT/pytest_parity.log 2>&1
timeout 600 python bench.py --no-cpu --no-dense --no-e2e > $OUT/bench_c3.json 2> $OUT/bench_c3.err
timeout 600 python bench.py --no-cpu --no-dense --no-e2e --config c2ref > $OUT/bench_c2ref.json 2> $OUT/bench_c2ref.err
