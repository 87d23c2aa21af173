# Final measurement set of the round on the final code (round 2, session 3, after the stage-1 and host-path changes)
OUT=gpurun_out/r2s3final2; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit,temperature.gpu --format=csv > $OUT/gpu.txt
timeout 1800 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > $OUT/bench_c3.json 2> $OUT/bench_c3.err
for a in 0.90 0.98; do timeout 600 python bench.py --alpha $a --no-cpu --no-dense --no-e2e > $OUT/bench_c3_a$a.json 2>> $OUT/bench_misc.err; done
timeout 600 python bench.py --config c2 --no-cpu > $OUT/bench_c2.json 2>> $OUT/bench_misc.err
timeout 600 python bench.py --config c4 --no-cpu > $OUT/bench_c4_r2.json 2>> $OUT/bench_misc.err
timeout 900 python bench.py --config c4 --chunk-n 77 --no-cpu --no-dense --no-e2e > $OUT/bench_c4_r10.json 2>> $OUT/bench_misc.err
timeout 900 python bench.py --config c2ref --no-cpu --no-e2e > $OUT/bench_c2ref.json 2>> $OUT/bench_misc.err
timeout 1500 python bench.py --config c3ref --no-cpu --no-e2e --no-dense > $OUT/bench_c3ref.json 2>> $OUT/bench_misc.err
timeout 1500 python bench.py --config c5 --steps 3 --no-cpu --no-dense --no-e2e > $OUT/bench_c5_1gpu.json 2>> $OUT/bench_misc.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $OUT/bench_reference.json 2>> $OUT/bench_misc.err
SA_DIST_BACKEND=gloo timeout 900 python bench.py --gpus 2 --config c3 --no-dense --no-cpu --no-e2e --steps 2 > $OUT/bench_c3_gpus2.json 2>> $OUT/bench_misc.err
SA_DIST_BACKEND=gloo timeout 900 python bench.py --gpus 2 --config c5 --no-dense --no-cpu --no-e2e --steps 1 --warmup 3 > $OUT/bench_c5_gpus2.json 2>> $OUT/bench_misc.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k1_|k2_|k3_|xf_|s1_|k_check|k_flag|k_pair|k_key|k_band|k_sampled" -c 200 --csv --log-file $OUT/launches_c3.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-dense --no-e2e > $OUT/ncu_bench.log 2>&1
ls -la $OUT
