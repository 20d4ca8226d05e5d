# LM head: masked row-block skipping — parity tests (incl. the skip case), timings on ragged RhoMath and Qwen.
timeout 600 python -m pytest tests/test_gpu_lmhead.py -q -x 2>&1 | tail -2
for mc in 1 3; do TBA_LM_MC=$mc timeout 300 python -m pytest tests/test_gpu_lmhead.py -q -x -k "skipped or ragged or tb_head" 2>&1 | tail -1; done
for w in rhomath qwen_shard pythia redteam; do
timeout 600 python bench.py --objective lmhead --workload $w --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); u=d['variants']['unfused_cublas_logits']
print('%-10s fused %.2f ms (%.0f useful TF/s, %s MHz)  paired: fused %.2f unfused %.2f matmul %.2f ratio %.3f' % (d['config']['workload'], d['ms_per_step'], d['roofline']['achieved'], d['clocks']['sm_mhz'], u['fused_ms_paired'], u['ms_per_step'], u['matmul_ms'], u['fused_over_unfused']))"
done
