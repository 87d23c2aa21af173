OUT=gpurun_out/r2au; mkdir -p $OUT
for r in "2,2,3,5" "1,1,2,3,5" "1,2,3,5" "2,3,5"; do echo "ramp $r" >> $OUT/e2e.txt; SA_HOST_RAMP=$r timeout 300 python tools/e2e_diag.py 2>&1 | grep "default\|one_lane" >> $OUT/e2e.txt; done
