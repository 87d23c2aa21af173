OUT=gpurun_out/r2g1; mkdir -p $OUT
timeout 120 ./tools/tmem_ld_bench > $OUT/tmem_ld_bench.txt 2>&1
timeout 600 python tools/guard_kinds.py 32768 1 2 ref > $OUT/guard_kinds_c2ref.txt 2>&1
