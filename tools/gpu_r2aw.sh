OUT=gpurun_out/r2aw; mkdir -p $OUT
timeout 600 compute-sanitizer --tool racecheck python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "large_logits and 2-2.5" > $OUT/racecheck_band.txt 2>&1
timeout 600 compute-sanitizer --tool synccheck python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "large_logits and 2-2.5" > $OUT/synccheck_band.txt 2>&1
timeout 600 compute-sanitizer --tool initcheck python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "large_logits and 2-2.5" > $OUT/initcheck_band.txt 2>&1
