OUT=gpurun_out/r2a; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv > $OUT/gpu.txt
nproc > $OUT/nproc.txt; lscpu | head -20 >> $OUT/nproc.txt
timeout 900 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.log 2>&1
timeout 600 python bench.py --no-cpu > $OUT/bench_c3.json 2> $OUT/bench_c3.err
python -c "import vllm.vllm_flash_attn as f; print(dir(f))" > $OUT/fa4_probe.txt 2>&1
python -c "from vllm.vllm_flash_attn.cute import interface as i; print(dir(i))" >> $OUT/fa4_probe.txt 2>&1
python -c "import flash_attn.cute as c; print(dir(c))" >> $OUT/fa4_probe.txt 2>&1
