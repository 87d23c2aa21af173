OUT=gpurun_out/r2u; mkdir -p $OUT
timeout 600 python tools/e2e_diag.py > $OUT/e2e_diag.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "streaming" > $OUT/pytest.log 2>&1
timeout 600 python bench.py --no-cpu --no-dense > $OUT/bench_c3.json 2> $OUT/bench_c3.err
