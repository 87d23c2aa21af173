OUT=gpurun_out/r2p; mkdir -p $OUT
( time timeout 900 python bench.py --config c2ref --no-cpu ) > $OUT/bench_c2ref.json 2> $OUT/bench_c2ref.err
( time timeout 1200 python bench.py --config c3ref --no-cpu --no-e2e ) > $OUT/bench_c3ref.json 2> $OUT/bench_c3ref.err
for a in 0.90 0.98; do timeout 900 python bench.py --config c2ref --alpha $a --no-cpu --no-e2e --no-dense > $OUT/bench_c2ref_a$a.json 2>> $OUT/bench_c2ref.err; done
