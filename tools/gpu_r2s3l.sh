# GPU suite + C3 / C4 lines on the K1 early-release + fold-batching build
OUT=gpurun_out/r2s3l; mkdir -p $OUT
timeout 1800 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.txt 2>&1
timeout 600 python bench.py --config c4 --chunk-n 77 --no-cpu --no-dense --no-e2e > $OUT/bench_c4_r10.json 2> $OUT/bench.err
timeout 600 python bench.py --config c4 --no-cpu --no-dense --no-e2e > $OUT/bench_c4_r2.json 2>> $OUT/bench.err
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu --no-dense > $OUT/bench_c3.json 2>> $OUT/bench.err
