# Full GPU suite at HEAD; A/B: one-warp-row forward with 1 of 8 pairs on the polynomial (n32e) vs 1 of 4
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -x 2>&1 | tail -3
python scripts/ab_variants.py n32e=TBA_FWD_NP32=-1 > /dev/null 2>&1
B="python bench.py --no-e2e --no-cpu-baseline --no-variants"
for rep in 1 2; do
for v in prod n32e; do
  if [ $v = prod ]; then L=""; else L="/tmp/tba_variants/$v/libtba.so"; fi
  for wl in pythia redteam gsm8k_t3 rhomath qwen_shard; do
  TBA_LIBRARY=$L $B --workload $wl > gpurun_out/n32_${v}_$wl.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/n32_${v}_$wl.json')); k=d['kernels']; print('$v', '$wl', round(d['ms_per_step'],4), 'fwd', round(k['fwd_ms'],4), round(k['fwd_frac'],3), 'bwd', round(k['bwd_ms'],4), 'step', round(k['step_frac'],3), d['clocks']['sm_mhz'])"
  done
done
done
