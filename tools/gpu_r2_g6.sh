OUT=gpurun_out/r2g6; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.txt 2>&1
timeout 600 python bench.py --config c2ref --no-cpu --no-e2e --no-dense > $OUT/bench_c2ref.json 2> $OUT/bench.err
timeout 600 python bench.py --no-cpu --no-e2e --no-dense > $OUT/bench_c3.json 2>> $OUT/bench.err
timeout 900 python bench.py --config c4 --chunk-n 77 --no-cpu --no-dense --no-e2e > $OUT/bench_c4_r10.json 2>> $OUT/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k1_|k2_|k3_|xf_|s1_|k_" -c 120 --csv --log-file $OUT/launches_c2ref.csv python bench.py --config c2ref --steps 1 --warmup 3 --no-cpu --no-dense --no-e2e > $OUT/ncu_bench.log 2>&1
