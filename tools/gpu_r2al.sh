OUT=gpurun_out/r2al; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "host_path_shapes or streaming" > $OUT/pytest.log 2>&1
