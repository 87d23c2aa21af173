OUT=gpurun_out/r2q; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden_metrics.py -m gpu -q -x > $OUT/pytest_parity.log 2>&1
timeout 600 python bench.py --no-cpu --no-dense > $OUT/bench_c3.json 2> $OUT/bench_c3.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file $OUT/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-dense --no-e2e > $OUT/ncu_bench.log 2>&1
