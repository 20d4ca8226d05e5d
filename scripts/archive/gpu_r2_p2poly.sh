# A/B: compile-time stash size (prod) vs runtime (rks); deferred pass 2 with the FMA-pipe exp2 on 1 of 4 (pp1) / 1 of 8 (pp2) element pairs vs none
mkdir -p gpurun_out
python scripts/ab_variants.py pp1=TBA_DEFER_P2POLY=1 pp2=TBA_DEFER_P2POLY=2 rks=TBA_AB_RUNTIME_KS > /dev/null 2>&1
timeout 900 python -m pytest -q -m gpu tests/test_gpu_fused.py tests/test_gpu_tbap.py tests/test_gpu_hostile.py -k "deferred or confident or token_regions" 2>&1 | tail -1
TBA_LIBRARY=/tmp/tba_variants/pp2/libtba.so timeout 900 python -m pytest -q -m gpu tests/test_gpu_fused.py tests/test_gpu_tbap.py tests/test_gpu_hostile.py -k "deferred or confident" 2>&1 | tail -1
for rep in 1 2; do
for v in prod rks pp1 pp2; do
  if [ $v = prod ]; then L=""; else L="/tmp/tba_variants/$v/libtba.so"; fi
  for wl in qwen_shard math_t5_shard rhomath; do
    TBA_LIBRARY=$L timeout 300 python bench.py --workload $wl --schedule deferred --no-e2e --no-cpu-baseline --no-variants > gpurun_out/pq_${v}_$wl.json 2>gpurun_out/pq_${v}_$wl.err
    python -c "
import json; d=json.load(open('gpurun_out/pq_${v}_$wl.json')); print('$v', '$wl', round(d['ms_per_step'],4), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])" || tail -3 gpurun_out/pq_${v}_$wl.err
  done
  TBA_LIBRARY=$L python scripts/microbench/defer_steps.py 2>/dev/null > gpurun_out/pq_steps_$v.txt; python -c "
for l in open('gpurun_out/pq_steps_$v.txt'):
    if 'sleep' in l:
        p=l.split(); t=sorted(map(float,p[3:])); print('$v', p[0], p[1], p[2], 'median', t[len(t)//2], 'min', t[0])
" 2>/dev/null | head -2
done
done
