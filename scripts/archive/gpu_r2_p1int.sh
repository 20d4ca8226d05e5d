# A/B: deferred pass 1 with 32-bit indices and a uniform token-iteration test (product candidate) vs the
# previous HEAD (ab_libs/headref: built from the stashed tree)
mkdir -p gpurun_out
timeout 900 python -m pytest -q -m gpu tests/test_gpu_fused.py tests/test_gpu_tbap.py tests/test_gpu_hostile.py tests/test_gpu_guard.py -k "deferred or confident or token_regions or bounds" 2>&1 | tail -1
for rep in 1 2; do
for v in prod headref; do
  if [ $v = prod ]; then L=""; else L="$PWD/ab_libs/$v/libtba.so"; fi
  for wl in qwen_shard math_t5_shard pythia_fp32; do
    TBA_LIBRARY=$L timeout 300 python bench.py --workload $wl --schedule deferred --no-e2e --no-cpu-baseline --no-variants > gpurun_out/pi_${v}_$wl.json 2>gpurun_out/pi_${v}_$wl.err
    python -c "
import json; d=json.load(open('gpurun_out/pi_${v}_$wl.json')); print('$v', '$wl', round(d['ms_per_step'],4), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])" 2>/dev/null || tail -2 gpurun_out/pi_${v}_$wl.err
  done
  TBA_LIBRARY=$L python scripts/microbench/defer_steps.py 2>/dev/null > gpurun_out/pi_steps_$v.txt; python -c "
for l in open('gpurun_out/pi_steps_$v.txt'):
    if 'sleep' in l:
        p=l.split(); t=sorted(map(float,p[3:])); print('$v', p[0], p[1], p[2], 'median', t[len(t)//2], 'min', t[0])
" 2>/dev/null | head -2
done
done
