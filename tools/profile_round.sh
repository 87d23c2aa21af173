#!/bin/bash
# One GPU session of evidence: GPU tests, bench lines (C3 full line with dense
# rows / e2e / CPU baseline, alpha sweep, C2, C4 at 2 % and 10 % sampling, C5 1M
# on one GPU), the ncu launch list of the C3 step and full captures of the hot
# kernels.  Writes into gpurun_out/$TAG/.
TAG=${1:-r1}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv > $OUT/gpu.txt
timeout 900 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1
timeout 900 python bench.py > $OUT/bench_c3.json 2> $OUT/bench_c3.err
for a in 0.90 0.98; do
  timeout 300 python bench.py --alpha $a --no-dense --no-cpu --no-e2e > $OUT/bench_c3_a$a.json 2>> $OUT/bench.err
done
timeout 300 python bench.py --config c2 --no-cpu > $OUT/bench_c2.json 2>> $OUT/bench.err
timeout 600 python bench.py --config c4 --no-cpu --no-e2e > $OUT/bench_c4_r2.json 2>> $OUT/bench.err
timeout 600 python bench.py --config c4 --chunk-n 77 --no-dense --no-cpu --no-e2e > $OUT/bench_c4_r10.json 2>> $OUT/bench.err
timeout 900 python bench.py --config c5 --steps 3 --no-dense --no-cpu --no-e2e > $OUT/bench_c5_1gpu.json 2>> $OUT/bench.err
timeout 600 python bench.py --impl reference > $OUT/bench_reference.json 2>> $OUT/bench.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
  timeout 300 python bench.py --steps 2 --warmup 3 --no-dense --no-cpu --no-e2e --no-graph > $OUT/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k3_share|k1_tc|k2_|xf_pass|s1_|k_check|k_flag" -s 0 -c 20 \
  -o $OUT/full timeout 600 python bench.py --steps 1 --warmup 3 --no-dense --no-cpu --no-e2e --no-graph > $OUT/ncu_full.log 2>&1
mkdir -p $OUT/sanitizer
for t in memcheck racecheck initcheck synccheck; do
  timeout 400 compute-sanitizer --tool $t python -c "import __graft_entry__ as g; g.smoke()" > $OUT/sanitizer/$t.txt 2>&1
done
ls -la $OUT
