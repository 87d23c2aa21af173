OUT=gpurun_out/r2n; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "schedule or graph or shards or short or gqa" > $OUT/pytest_sched.log 2>&1
timeout 600 python bench.py --no-cpu --no-dense > $OUT/bench_c3.json 2> $OUT/bench_c3.err
timeout 600 python bench.py --no-cpu --no-dense --config c2 > $OUT/bench_c2.json 2> $OUT/bench_c2.err
