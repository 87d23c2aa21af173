OUT=gpurun_out/r2s3g; mkdir -p $OUT
timeout 900 python tools/zero_block_stats.py --config c3 --heads 0 17 31 > $OUT/zero_blocks_c3.txt 2>&1
timeout 900 python tools/zero_block_stats.py --config c3 --heads 0 --gap 20 >> $OUT/zero_blocks_c3.txt 2>&1
