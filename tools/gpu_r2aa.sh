OUT=gpurun_out/r2aa; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "streaming or nonfinite" > $OUT/pytest.log 2>&1
timeout 600 python tools/e2e_diag.py > $OUT/e2e_diag.txt 2>&1
timeout 600 python tools/e2e_trace.py > $OUT/e2e_trace.txt 2>&1
