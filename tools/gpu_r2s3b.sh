# ncu evidence on the current code: K1 at C4 10 % with source (stall map), K3 at C3 (DRAM traffic per launch)
OUT=gpurun_out/r2s3b; mkdir -p $OUT
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k1_tc" -s 2 -c 1 -o $OUT/k1_c4_77 \
  python tools/stage1_bench.py --config c4 --chunk-n 77 --reps 1 > $OUT/ncu_k1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k3_share" -s 3 -c 1 -o $OUT/k3_c3 \
  python bench.py --steps 1 --warmup 3 --no-dense --no-cpu --no-e2e --no-graph > $OUT/ncu_k3.log 2>&1
ls -la $OUT
