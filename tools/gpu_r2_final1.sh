OUT=gpurun_out/r2f1; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit,temperature.gpu --format=csv > $OUT/gpu.txt
timeout 900 python bench.py > $OUT/bench_c3.json 2> $OUT/bench_c3.err
for a in 0.90 0.98; do timeout 600 python bench.py --alpha $a --no-cpu --no-dense --no-e2e > $OUT/bench_c3_a$a.json 2>> $OUT/bench_misc.err; done
timeout 600 python bench.py --config c2 --no-cpu > $OUT/bench_c2.json 2>> $OUT/bench_misc.err
timeout 600 python bench.py --config c4 --no-cpu > $OUT/bench_c4_r2.json 2>> $OUT/bench_misc.err
timeout 900 python bench.py --config c4 --chunk-n 77 --no-cpu --no-dense --no-e2e > $OUT/bench_c4_r10.json 2>> $OUT/bench_misc.err
timeout 1500 python bench.py --config c5 --steps 3 --no-cpu --no-dense --no-e2e > $OUT/bench_c5_1gpu.json 2>> $OUT/bench_misc.err
timeout 900 python bench.py --impl reference > $OUT/bench_reference.json 2>> $OUT/bench_misc.err
