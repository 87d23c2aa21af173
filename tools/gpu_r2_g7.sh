OUT=gpurun_out/r2g7; mkdir -p $OUT
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"xf_" -s 0 -c 2 -o $OUT/xf_full python bench.py --config c2ref --steps 1 --warmup 1 --no-cpu --no-dense --no-e2e > $OUT/ncu.log 2>&1
