# GPU suite + smoke + C3 / C4 10 % lines on the final K1
OUT=gpurun_out/r2s3v; mkdir -p $OUT
timeout 1800 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1
timeout 600 python bench.py --config c4 --chunk-n 77 --no-cpu --no-dense --no-e2e > $OUT/bench_c4_r10.json 2> $OUT/bench.err
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu > $OUT/bench_c3.json 2>> $OUT/bench.err
