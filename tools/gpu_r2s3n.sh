# sanitizers on the session-3 code: smoke (all tools), the stage-1 / guard tests (memcheck, racecheck, synccheck), the p2p peer-store kernel (memcheck)
OUT=gpurun_out/r2s3n; mkdir -p $OUT/sanitizer
for t in memcheck racecheck initcheck synccheck; do
  timeout 600 compute-sanitizer --tool $t python -c "import __graft_entry__ as g; g.smoke()" > $OUT/sanitizer/smoke_$t.txt 2>&1
done
timeout 1500 compute-sanitizer --tool memcheck python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "golden or guard or kat or stage1 or block_reduce" > $OUT/sanitizer/memcheck_parity_subset.txt 2>&1
timeout 900 compute-sanitizer --tool racecheck python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "golden_case" > $OUT/sanitizer/racecheck_golden.txt 2>&1
timeout 900 compute-sanitizer --tool synccheck python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "golden_case" > $OUT/sanitizer/synccheck_golden.txt 2>&1
timeout 900 compute-sanitizer --tool memcheck python -c "
import torch, paper_2406_15486_b200 as sa
from paper_2406_15486_b200 import synth
q, k, v, _ = synth.make_inputs(4096, 4, 2, seed=1, device='cuda')
peer = torch.zeros_like(q); out = torch.empty_like(q)
o, r = sa.sample_attention(q, k, v, alpha=0.95, chunk_n=2, out=out, peer_out=[peer.data_ptr()])
torch.cuda.synchronize()
assert torch.equal(out, peer), 'peer copy differs'
print('peer-store memcheck run ok')
" > $OUT/sanitizer/memcheck_peer_store.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k1_tc" -s 2 -c 1 -o $OUT/k1_c4_77_final python tools/stage1_bench.py --config c4 --chunk-n 77 --reps 1 > $OUT/ncu_k1.log 2>&1
for f in $OUT/sanitizer/*.txt; do echo "== $f"; grep -E "ERROR SUMMARY|passed|failed|ok" $f | tail -3; done
