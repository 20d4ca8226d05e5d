# A/B: deferred pass 2 L2 part in forward order (fwd2) vs from the end (product); the max shared-memory
# carveout with larger stashes (coNNN)
mkdir -p gpurun_out
python scripts/ab_variants.py fwd2=TBA_DEFER_P2FWD co96=TBA_DEFER_CARVEOUT=1 co104=TBA_DEFER_CARVEOUT=1,TBA_DEFER_STASH_KB=104 co108=TBA_DEFER_CARVEOUT=1,TBA_DEFER_STASH_KB=108 co110=TBA_DEFER_CARVEOUT=1,TBA_DEFER_STASH_KB=110 fwdco108=TBA_DEFER_P2FWD,TBA_DEFER_CARVEOUT=1,TBA_DEFER_STASH_KB=108 > /dev/null 2>&1
for v in fwd2 co108; do
TBA_LIBRARY=/tmp/tba_variants/$v/libtba.so timeout 900 python -m pytest -q -m gpu tests/test_gpu_fused.py tests/test_gpu_tbap.py tests/test_gpu_hostile.py -k "deferred or confident" 2>&1 | tail -1
done
for rep in 1 2; do
for v in prod fwd2 co96 co104 co108 co110 fwdco108; do
  if [ $v = prod ]; then L=""; else L="/tmp/tba_variants/$v/libtba.so"; fi
  for wl in qwen_shard math_t5_shard; do
    TBA_LIBRARY=$L timeout 300 python bench.py --workload $wl --schedule deferred --no-e2e --no-cpu-baseline --no-variants > gpurun_out/or_${v}_$wl.json 2>gpurun_out/or_${v}_$wl.err
    python -c "
import json; d=json.load(open('gpurun_out/or_${v}_$wl.json')); print('$v', '$wl', round(d['ms_per_step'],4), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])" || tail -3 gpurun_out/or_${v}_$wl.err
  done
  TBA_LIBRARY=$L python scripts/microbench/defer_steps.py 2>&1 | python -c "
import sys
for l in sys.stdin:
    if 'sleep' in l:
        p=l.split(); t=sorted(map(float,p[3:])); print('$v', p[0], p[1], p[2], 'median', t[len(t)//2], 'min', t[0])
" | head -2
  if [ $rep = 1 ]; then
  TBA_LIBRARY=$L ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:row_single -s 3 -c 1 --csv python bench.py --no-e2e --no-cpu-baseline --no-variants --workload qwen_group --schedule deferred --steps 1 --warmup 3 2>/dev/null | grep -E "dram__|gpu__time|warps_active" | awk -F'","' -v v=$v '{print v, $(NF-2), $NF}'
  fi
done
done
