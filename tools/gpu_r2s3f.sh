# launch list of the C4 10 % step (stage-1 / stage-2 kernel shares)
OUT=gpurun_out/r2s3f; mkdir -p $OUT
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k1_|k2_|k3_|xf_|s1_|k_check|k_flag|k_pair|k_key|k_band|k_sampled" -c 200 --csv --log-file $OUT/launches_c4_77.csv python bench.py --config c4 --chunk-n 77 --steps 1 --warmup 3 --no-cpu --no-dense --no-e2e --no-graph > $OUT/ncu_bench.log 2>&1
