OUT=gpurun_out/r2s3t; mkdir -p $OUT
REPS=12 timeout 1500 python tools/e2e_ramp_ab.py 1,1,2,3,5/1,2,3 1,1,2,3,5/1,1,2 1,1,2,3,5/1,1,2,3 > $OUT/e2e_tail_ab.txt 2>&1
REPS=12 timeout 1500 python tools/e2e_ramp_ab.py 1,1,2,3,5/1,1,2,3 1,1,2,3,5/1,1,2 1,1,2,3,5/1,2,3 >> $OUT/e2e_tail_ab.txt 2>&1
