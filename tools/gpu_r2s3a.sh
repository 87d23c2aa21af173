OUT=gpurun_out/r2s3a; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit,temperature.gpu --format=csv > $OUT/gpu.txt
timeout 1800 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu > $OUT/bench_c3.json 2> $OUT/bench_c3.err
