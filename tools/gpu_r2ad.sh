OUT=gpurun_out/r2ad; mkdir -p $OUT
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k1_tc|xf_pass" -s 2 -c 2 -o $OUT/k1_c4 python bench.py --config c4 --chunk-n 77 --steps 1 --warmup 3 --no-cpu --no-dense --no-e2e --no-graph > $OUT/ncu.log 2>&1
