OUT=gpurun_out/r2x; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.log 2>&1
timeout 600 python bench.py --no-cpu --no-dense > $OUT/bench_c3.json 2> $OUT/bench_c3.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k1_|k2_|k3_|xf_|s1_|k_check|k_flag|k_pair|k_key|k_sampled" -c 200 --csv --log-file $OUT/launches_c3.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-dense --no-e2e > $OUT/ncu_bench.log 2>&1
