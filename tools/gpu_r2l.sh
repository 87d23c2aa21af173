OUT=gpurun_out/r2l; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x > $OUT/pytest_parity.log 2>&1
timeout 300 python tools/dump_mask.py --config c3 --alpha 0.95 --out $OUT/mask_c3.npz > $OUT/dump.log 2>&1
timeout 300 python tools/dump_mask.py --config c2 --alpha 0.95 --out $OUT/mask_c2.npz >> $OUT/dump.log 2>&1
timeout 300 python tools/dump_mask.py --config c4 --alpha 0.95 --out $OUT/mask_c4.npz >> $OUT/dump.log 2>&1
SA_LIB_PATH=variants/lib_prof.so timeout 300 python tools/k3_profile.py > $OUT/k3_profile_c3.txt 2>&1
SA_LIB_PATH=variants/lib_prof.so timeout 300 python tools/k3_profile.py --dense > $OUT/k3_profile_dense.txt 2>&1
