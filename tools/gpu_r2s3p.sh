# K3 epilogue staged through smem (whole-row coalesced stores) vs row-per-thread 16-byte stores; GPU tests on the staged build
OUT=gpurun_out/r2s3p; mkdir -p $OUT
L="variants/lib_k3epi0.so variants/lib_k3epi1.so"
timeout 900 python tools/k3_ab.py --libs $L --reps 16 > $OUT/k3epi_c3.txt 2>&1
timeout 900 python tools/k3_ab.py --libs variants/lib_k3epi1.so variants/lib_k3epi0.so --reps 16 >> $OUT/k3epi_c3.txt 2>&1
timeout 900 python tools/k3_ab.py --libs $L --reps 16 --config c2 > $OUT/k3epi_c2.txt 2>&1
timeout 900 python tools/k3_ab.py --libs $L --reps 4 --dense > $OUT/k3epi_dense.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.txt 2>&1
