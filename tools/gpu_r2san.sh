OUT=gpurun_out/r2san; mkdir -p $OUT
for t in memcheck racecheck initcheck synccheck; do
  timeout 500 compute-sanitizer --tool $t python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$t.txt 2>&1
done
timeout 1500 compute-sanitizer --tool memcheck python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "schedule or streaming or guard or nonfinite or case or shards" > $OUT/memcheck_gpu_tests.txt 2>&1
timeout 1200 compute-sanitizer --tool racecheck python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "schedule_overlap_pairing and 12" > $OUT/racecheck_pairing.txt 2>&1
timeout 1200 compute-sanitizer --tool synccheck python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "schedule_overlap_pairing and 12 or guard_policies" > $OUT/synccheck_tests.txt 2>&1
