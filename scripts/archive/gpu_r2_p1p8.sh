# Output-guard tests; A/B: deferred pass 1 with 1 of 8 pairs on the FMA-pipe exp2 (p1p8); the Qwen-row
# forward with 1 of 8 (f8) instead of 1 of 4 pairs
mkdir -p gpurun_out
timeout 900 python -m pytest -q -m gpu tests/test_gpu_guard.py 2>&1 | tail -3
python scripts/ab_variants.py p1p8=TBA_DEFER_NP1=-1 f8=TBA_FWD_NP64=-1 > /dev/null 2>&1
TBA_LIBRARY=/tmp/tba_variants/p1p8/libtba.so timeout 900 python -m pytest -q -m gpu tests/test_gpu_fused.py -k "deferred or token_regions" 2>&1 | tail -1
TBA_LIBRARY=/tmp/tba_variants/f8/libtba.so timeout 900 python -m pytest -q -m gpu tests/test_gpu_parity.py tests/test_gpu_hostile.py 2>&1 | tail -1
for rep in 1 2; do
for v in prod p1p8; do
  if [ $v = prod ]; then L=""; else L="/tmp/tba_variants/$v/libtba.so"; fi
  for wl in qwen_shard math_t5_shard; do
    TBA_LIBRARY=$L timeout 300 python bench.py --workload $wl --schedule deferred --no-e2e --no-cpu-baseline --no-variants > gpurun_out/p18_${v}_$wl.json 2>/dev/null
    python -c "
import json; d=json.load(open('gpurun_out/p18_${v}_$wl.json')); print('$v', '$wl', round(d['ms_per_step'],4), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])"
  done
  TBA_LIBRARY=$L python scripts/microbench/defer_steps.py 2>/dev/null > gpurun_out/p18_steps_$v.txt; python -c "
for l in open('gpurun_out/p18_steps_$v.txt'):
    if 'sleep' in l:
        p=l.split(); t=sorted(map(float,p[3:])); print('$v', p[0], p[1], p[2], 'median', t[len(t)//2], 'min', t[0])
" 2>/dev/null | head -2
done
for v in prod f8; do
  if [ $v = prod ]; then L=""; else L="/tmp/tba_variants/$v/libtba.so"; fi
  for wl in qwen_shard math_t5_shard; do
  TBA_LIBRARY=$L python bench.py --no-e2e --no-cpu-baseline --no-variants --workload $wl > gpurun_out/f8_${v}_$wl.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/f8_${v}_$wl.json')); k=d['kernels']; print('$v', '$wl', round(d['ms_per_step'],4), 'fwd', round(k['fwd_ms'],4), round(k['fwd_frac'],3), 'bwd', round(k['bwd_ms'],4), 'step', round(k['step_frac'],3), d['clocks']['sm_mhz'])"
  done
done
done
