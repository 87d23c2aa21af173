OUT=gpurun_out/r2ar; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.log 2>&1
timeout 300 python tools/guard_diag.py 131072 1 > $OUT/guard_c3.txt 2>&1
timeout 300 python tools/guard_diag.py 98304 77 > $OUT/guard_c4_77.txt 2>&1
timeout 300 python tools/guard_large_logits.py > $OUT/guard_large.txt 2>&1
timeout 300 python tools/rownorm_diag.py 98304 77 8 > $OUT/rn_c4_77.txt 2>&1
