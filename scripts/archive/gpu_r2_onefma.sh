# A/B: deferred pass 2 forming the exponent with one FFMA2 for bf16 G (onefma) vs FFMA2 + FADD2 (product)
mkdir -p gpurun_out
TBA_LIBRARY=$PWD/ab_libs/onefma/libtba.so timeout 900 python -m pytest -q -m gpu tests/test_gpu_fused.py tests/test_gpu_tbap.py tests/test_gpu_hostile.py tests/test_gpu_guard.py -k "deferred or confident or token_regions or bounds" 2>&1 | tail -3
for rep in 1 2; do
for v in prod onefma; do
  if [ $v = prod ]; then L=""; else L="$PWD/ab_libs/$v/libtba.so"; fi
  for wl in qwen_shard math_t5_shard rhomath; do
    TBA_LIBRARY=$L timeout 300 python bench.py --workload $wl --schedule deferred --no-e2e --no-cpu-baseline --no-variants > gpurun_out/of_${v}_$wl.json 2>gpurun_out/of_${v}_$wl.err
    python -c "
import json; d=json.load(open('gpurun_out/of_${v}_$wl.json')); print('$v', '$wl', round(d['ms_per_step'],4), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])" 2>/dev/null || tail -2 gpurun_out/of_${v}_$wl.err
  done
  TBA_LIBRARY=$L python scripts/microbench/defer_steps.py 2>/dev/null > gpurun_out/of_steps_$v.txt; python -c "
for l in open('gpurun_out/of_steps_$v.txt'):
    if 'sleep' in l:
        p=l.split(); t=sorted(map(float,p[3:])); print('$v', p[0], p[1], p[2], 'median', t[len(t)//2], 'min', t[0])
" 2>/dev/null | head -2
done
done
