OUT=gpurun_out/r2bc; mkdir -p $OUT
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k1_tc|xf_items|k_band_scores|k2_select|k2_pair|s1_fold|k2_merge" -s 10 -c 8 -o $OUT/stage12_c4 python bench.py --config c4 --chunk-n 77 --steps 1 --warmup 3 --no-cpu --no-dense --no-e2e --no-graph > $OUT/ncu_c4.log 2>&1
