OUT=gpurun_out/r2b; mkdir -p $OUT
free -g > $OUT/mem.txt
timeout 1500 python -m pytest tests -m gpu -q -rA --durations=25 > $OUT/pytest_gpu.log 2>&1
timeout 600 python bench.py > $OUT/bench_c3.json 2> $OUT/bench_c3.err
SA_DIST_BACKEND=gloo timeout 600 python bench.py --gpus 2 --no-dense --no-cpu --no-e2e --steps 3 > $OUT/bench_c3_gpus2.json 2> $OUT/bench_c3_gpus2.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
