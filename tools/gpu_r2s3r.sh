OUT=gpurun_out/r2s3r; mkdir -p $OUT
REPS=16 timeout 1200 python tools/e2e_ramp_ab.py 2,2,3,5 1,1,2,3,5 > $OUT/e2e_ramp_ab2.txt 2>&1
REPS=16 timeout 1200 python tools/e2e_ramp_ab.py 1,1,2,3,5 2,2,3,5 >> $OUT/e2e_ramp_ab2.txt 2>&1
