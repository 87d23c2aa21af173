OUT=gpurun_out/r2g10; mkdir -p $OUT
timeout 900 python bench.py --config c3ref --no-cpu --no-e2e > $OUT/bench_c3ref.json 2> $OUT/bench.err
timeout 600 python bench.py --config c2ref --alpha 0.90 --no-cpu --no-e2e --no-dense > $OUT/bench_c2ref_a0.90.json 2>> $OUT/bench.err
timeout 1500 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.txt 2>&1
timeout 600 python bench.py --no-cpu --no-e2e --no-dense > $OUT/bench_c3.json 2>> $OUT/bench.err
timeout 900 python bench.py --config c4 --chunk-n 77 --no-cpu --no-dense --no-e2e > $OUT/bench_c4_r10.json 2>> $OUT/bench.err
timeout 600 python bench.py --config c2ref --no-cpu --no-e2e --no-dense > $OUT/bench_c2ref.json 2>> $OUT/bench.err
