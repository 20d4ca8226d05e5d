# A/B: persistent warp-per-row forward with next-row prefetch (persist) vs one-shot CTAs of 8 rows
mkdir -p gpurun_out
python scripts/ab_variants.py persist=TBA_FWD_PERSIST > /dev/null 2>&1
TBA_LIBRARY=/tmp/tba_variants/persist/libtba.so timeout 1200 python -m pytest -q -m gpu tests/test_gpu_parity.py tests/test_gpu_fused.py tests/test_gpu_hostile.py tests/test_gpu_variants.py 2>&1 | tail -2
B="python bench.py --no-e2e --no-cpu-baseline --no-variants"
for rep in 1 2; do
for v in prod persist; do
  if [ $v = prod ]; then L=""; else L="/tmp/tba_variants/$v/libtba.so"; fi
  for wl in pythia redteam gsm8k_t3 gsm8k_k40 rhomath tldr_t4; do
  TBA_LIBRARY=$L $B --workload $wl > gpurun_out/ps_${v}_$wl.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/ps_${v}_$wl.json')); k=d['kernels']; print('$v', '$wl', round(d['ms_per_step'],4), 'fwd', round(k['fwd_ms'],4), round(k['fwd_frac'],3), 'bwd', round(k['bwd_ms'],4), 'step', round(k['step_frac'],3), d['clocks']['sm_mhz'])"
  done
done
done
