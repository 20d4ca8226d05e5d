# LM head epilogue change: parity tests, then the paired fused-vs-cuBLAS ratio (box-independent).
timeout 600 python -m pytest tests/test_gpu_lmhead.py -q -x 2>&1 | tail -2
timeout 120 python scripts/lmhead_debug.py 2>&1 | tail -6
for rep in 1 2; do
timeout 600 python bench.py --objective lmhead --steps 12 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); u=d['variants']['unfused_cublas_logits']
print('fused %.2f ms (%.0f TF/s, %s MHz)  paired: fused %.2f unfused %.2f matmul %.2f ratio %.3f' % (d['ms_per_step'], d['roofline']['achieved'], d['clocks']['sm_mhz'], u['fused_ms_paired'], u['ms_per_step'], u['matmul_ms'], u['fused_over_unfused']))"
done
