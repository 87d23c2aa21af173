OUT=gpurun_out/r2s3q; mkdir -p $OUT
timeout 900 python tools/e2e_ramp_ab.py > $OUT/e2e_ramp_ab.txt 2>&1
