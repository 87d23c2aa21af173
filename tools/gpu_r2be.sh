OUT=gpurun_out/r2be; mkdir -p $OUT
timeout 1500 compute-sanitizer --tool memcheck python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden_metrics.py -m gpu -q -x > $OUT/memcheck_gpu_tests.txt 2>&1
SA_DIST_BACKEND=gloo timeout 900 python bench.py --gpus 2 --config c3 --no-dense --no-cpu --no-e2e --steps 2 > $OUT/bench_c3_gpus2.json 2> $OUT/bench_c3_gpus2.err
SA_DIST_BACKEND=gloo timeout 900 python bench.py --gpus 2 --config c5 --no-dense --no-cpu --no-e2e --steps 1 --warmup 3 > $OUT/bench_c5_gpus2.json 2> $OUT/bench_c5_gpus2.err
