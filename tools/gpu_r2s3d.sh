# the output gather fused into stage 3 (p2p): two-rank test on one GPU, 2-rank C5 bench through it, K3 A/B vs the pre-p2p build
OUT=gpurun_out/r2s3d; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_p2p_gather.py -q -x > $OUT/pytest_p2p.txt 2>&1
timeout 900 python tools/k3_ab.py --libs variants/lib_pre_p2p.so variants/lib_p2p.so --reps 16 > $OUT/k3_p2p_ab.txt 2>&1
SA_DIST_BACKEND=gloo timeout 900 python bench.py --gpus 2 --config c5 --no-dense --no-cpu --no-e2e --steps 1 --warmup 3 > $OUT/bench_c5_gpus2_p2p.json 2> $OUT/bench_c5_gpus2_p2p.err
timeout 1800 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.txt 2>&1
