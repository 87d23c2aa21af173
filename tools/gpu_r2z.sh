OUT=gpurun_out/r2z; mkdir -p $OUT
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"k3_share" -s 1 -c 1 -o $OUT/k3_full python bench.py --steps 1 --warmup 3 --no-cpu --no-dense --no-e2e --no-graph > $OUT/ncu_k3.log 2>&1
