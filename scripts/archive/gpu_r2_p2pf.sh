# A/B: L2 bulk prefetch of the deferred pass 2's L2 part at the start of pass 2 (p2pf); pass-2 unroll 6 / 12
mkdir -p gpurun_out
python scripts/ab_variants.py p2pf=TBA_DEFER_P2PF > /dev/null 2>&1
TBA_LIBRARY=/tmp/tba_variants/p2pf/libtba.so timeout 900 python -m pytest -q -m gpu tests/test_gpu_fused.py tests/test_gpu_tbap.py -k "deferred" 2>&1 | tail -1
for rep in 1 2; do
for v in prod p2pf; do
  if [ $v = prod ]; then L=""; else L="/tmp/tba_variants/$v/libtba.so"; fi
  for wl in qwen_shard math_t5_shard; do
    TBA_LIBRARY=$L timeout 300 python bench.py --workload $wl --schedule deferred --no-e2e --no-cpu-baseline --no-variants > gpurun_out/pp_${v}_$wl.json 2>gpurun_out/pp_${v}_$wl.err
    python -c "
import json; d=json.load(open('gpurun_out/pp_${v}_$wl.json')); print('$v', '$wl', round(d['ms_per_step'],4), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])" || tail -3 gpurun_out/pp_${v}_$wl.err
  done
  TBA_LIBRARY=$L python scripts/microbench/defer_steps.py 2>/dev/null > gpurun_out/pp_steps_$v.txt; python -c "
for l in open('gpurun_out/pp_steps_$v.txt'):
    if 'sleep' in l:
        p=l.split(); t=sorted(map(float,p[3:])); print('$v', p[0], p[1], p[2], 'median', t[len(t)//2], 'min', t[0])
" | head -2
  if [ $rep = 1 ]; then
  TBA_LIBRARY=$L ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum --clock-control none -k regex:row_single -s 3 -c 1 --csv python bench.py --no-e2e --no-cpu-baseline --no-variants --workload qwen_group --schedule deferred --steps 1 --warmup 3 2>/dev/null | grep -E "dram__|gpu__time" | awk -F'","' -v v=$v '{print v, $(NF-2), $NF}'
  fi
done
done
