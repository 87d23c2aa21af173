OUT=gpurun_out/r2av; mkdir -p $OUT
timeout 300 python tools/k3_overhead.py > $OUT/overhead.txt 2>&1
