OUT=gpurun_out/r2g2; mkdir -p $OUT
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k1_|k2_|k3_|xf_|s1_|k_check|k_flag|k_pair|k_key|k_sampled|k_band|k_" -c 120 --csv --log-file $OUT/launches_c2ref.csv python bench.py --config c2ref --steps 1 --warmup 3 --no-cpu --no-dense --no-e2e > $OUT/ncu_bench.log 2>&1
