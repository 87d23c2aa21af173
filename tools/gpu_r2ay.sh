OUT=gpurun_out/r2ay; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.log 2>&1
timeout 300 python bench.py --no-cpu --no-dense --no-e2e > $OUT/bench_c3.json 2> $OUT/bench.err
timeout 300 python bench.py --config c4 --chunk-n 77 --no-cpu --no-dense --no-e2e > $OUT/bench_c4_r10.json 2>> $OUT/bench.err
timeout 300 python bench.py --config c4 --no-cpu --no-dense --no-e2e > $OUT/bench_c4.json 2>> $OUT/bench.err
timeout 300 python bench.py --config c2ref --no-cpu --no-dense --no-e2e > $OUT/bench_c2ref.json 2>> $OUT/bench.err
timeout 600 python bench.py --config c3ref --no-cpu --no-dense --no-e2e > $OUT/bench_c3ref.json 2>> $OUT/bench.err
timeout 600 compute-sanitizer --tool memcheck python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "guard or case" > $OUT/memcheck.txt 2>&1
