OUT=gpurun_out/r2s; mkdir -p $OUT
timeout 600 python tools/e2e_trace.py > $OUT/e2e_trace.txt 2>&1
timeout 600 python tools/e2e_trace.py '{"_lanes": 1}' > $OUT/e2e_trace_1lane.txt 2>&1
