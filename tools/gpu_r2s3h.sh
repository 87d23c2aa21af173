OUT=gpurun_out/r2s3h; mkdir -p $OUT
timeout 900 python tools/k1_dead_blocks.py --config c4 --chunk-n 77 > $OUT/k1_dead_c4_77.txt 2>&1
timeout 900 python tools/k1_dead_blocks.py --config c3 --chunk-n 1 --heads 0 17 --kpc 4 > $OUT/k1_dead_c3.txt 2>&1
