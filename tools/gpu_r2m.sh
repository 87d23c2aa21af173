OUT=gpurun_out/r2m; mkdir -p $OUT
L="variants/lib_qpf0.so variants/lib_qpf1.so variants/lib_qpf2.so"
timeout 900 python tools/k3_order_ab.py --libs $L --reps 8 > $OUT/order_ab_c3.txt 2>&1
timeout 600 python tools/k3_order_ab.py --libs $L --reps 8 --config c2 > $OUT/order_ab_c2.txt 2>&1
