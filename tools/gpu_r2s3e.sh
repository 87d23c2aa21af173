# K3 ring depth: K/V stages 2/2 (product) vs 3/2 vs 2/3, interleaved in-process A/B (C3, C3 dense, C2), two orders
OUT=gpurun_out/r2s3e; mkdir -p $OUT
L="variants/lib_k3_k2v2.so variants/lib_k3_k3v2.so variants/lib_k3_k2v3.so"
R="variants/lib_k3_k2v3.so variants/lib_k3_k3v2.so variants/lib_k3_k2v2.so"
timeout 900 python tools/k3_ab.py --libs $L --reps 16 > $OUT/k3_ring_c3.txt 2>&1
timeout 900 python tools/k3_ab.py --libs $R --reps 16 >> $OUT/k3_ring_c3.txt 2>&1
timeout 900 python tools/k3_ab.py --libs $L --reps 6 --dense > $OUT/k3_ring_dense.txt 2>&1
timeout 900 python tools/k3_ab.py --libs $L --reps 16 --config c2 > $OUT/k3_ring_c2.txt 2>&1
