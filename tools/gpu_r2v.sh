OUT=gpurun_out/r2v; mkdir -p $OUT
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k1_|k2_|k3_|xf_|s1_|k_check|k_flag|k_pair|k_key|k_sampled" -c 200 --csv --log-file $OUT/launches_c3.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-dense --no-e2e > $OUT/ncu_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"xf_pass|k1_tc|s1_fold|k2_select" -s 8 -c 4 -o $OUT/stage12 python bench.py --steps 1 --warmup 3 --no-cpu --no-dense --no-e2e > $OUT/ncu_full.log 2>&1
