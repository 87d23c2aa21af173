OUT=gpurun_out/r2j; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.log 2>&1
timeout 600 python bench.py --no-cpu > $OUT/bench_c3.json 2> $OUT/bench_c3.err
SA_LIB_PATH=variants/lib_prof.so timeout 300 python tools/k3_profile.py > $OUT/k3_profile_c3.txt 2>&1
SA_LIB_PATH=variants/lib_prof.so timeout 300 python tools/k3_profile.py --dense > $OUT/k3_profile_dense.txt 2>&1
