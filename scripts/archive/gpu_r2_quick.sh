# Quick check: hostile + fused/parity tests, default bench line, small-shape bench lines.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu -x tests/test_gpu_hostile.py tests/test_gpu_parity.py tests/test_gpu_fused.py tests/test_gpu_pipelined.py tests/test_gpu_tbap.py tests/test_gpu_variants.py 2>&1 | tail -4
for wl in qwen_shard pythia redteam gsm8k_t3 gsm8k_k40 tldr_t4 rhomath; do
  timeout 600 python bench.py --workload $wl --no-e2e --no-cpu-baseline > gpurun_out/q_$wl.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/q_$wl.json')); k=d['kernels']
print('$wl', round(d['ms_per_step'],4), 'fwd', round(k['fwd_ms'],4), round(k['fwd_frac'],3), 'bwd', round(k['bwd_ms'],4), round(d['roofline']['frac'],3), 'step', round(k['step_frac'],3), 'defer', round(d['variants']['deferred_scale']['ms_per_step'],4), d['clocks']['sm_mhz'])"
done
