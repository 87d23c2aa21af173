OUT=gpurun_out/r2ag; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "graph or shards or nonfinite" > $OUT/pytest.log 2>&1
timeout 600 python bench.py --no-cpu --no-dense --no-e2e > $OUT/bench_c3.json 2> $OUT/bench_c3.err
timeout 600 python bench.py --no-cpu --no-dense --no-e2e --config c4 > $OUT/bench_c4.json 2>> $OUT/bench_c3.err
timeout 900 python bench.py --no-cpu --no-dense --no-e2e --config c4 --chunk-n 77 > $OUT/bench_c4_r10.json 2>> $OUT/bench_c3.err
timeout 600 python bench.py --no-cpu --no-dense --no-e2e --config c2 > $OUT/bench_c2.json 2>> $OUT/bench_c3.err
