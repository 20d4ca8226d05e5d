# A/B: deferred pass with one 1024-thread CTA per SM per row and a 192 / 200 KB stash (bigNNN) vs
# two 512-thread CTAs with 96 KB each (the product)
mkdir -p gpurun_out
python scripts/ab_variants.py big192=TBA_DEFER_NT=1024,TBA_DEFER_STASH_KB=192 big200=TBA_DEFER_NT=1024,TBA_DEFER_STASH_KB=200 big192u4=TBA_DEFER_NT=1024,TBA_DEFER_STASH_KB=192,TBA_DEFER_U2=4 > /dev/null 2>&1
TBA_LIBRARY=/tmp/tba_variants/big192/libtba.so timeout 900 python -m pytest -q -m gpu tests/test_gpu_fused.py tests/test_gpu_tbap.py -k "deferred" 2>&1 | tail -1
for rep in 1 2; do
for v in prod big192 big200 big192u4; do
  if [ $v = prod ]; then L=""; else L="/tmp/tba_variants/$v/libtba.so"; fi
  for wl in qwen_shard math_t5_shard; do
    TBA_LIBRARY=$L timeout 300 python bench.py --workload $wl --schedule deferred --no-e2e --no-cpu-baseline --no-variants > gpurun_out/bg_${v}_$wl.json 2>gpurun_out/bg_${v}_$wl.err
    python -c "
import json; d=json.load(open('gpurun_out/bg_${v}_$wl.json')); print('$v', '$wl', round(d['ms_per_step'],4), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])" || tail -3 gpurun_out/bg_${v}_$wl.err
  done
  TBA_LIBRARY=$L python scripts/microbench/defer_steps.py 2>/dev/null > gpurun_out/bg_steps_$v.txt; python -c "
for l in open('gpurun_out/bg_steps_$v.txt'):
    if 'sleep' in l:
        p=l.split(); t=sorted(map(float,p[3:])); print('$v', p[0], p[1], p[2], 'median', t[len(t)//2], 'min', t[0])
" 2>/dev/null | head -2
  if [ $rep = 1 ]; then
  TBA_LIBRARY=$L ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum --clock-control none -k regex:row_single -s 3 -c 1 --csv python bench.py --no-e2e --no-cpu-baseline --no-variants --workload qwen_group --schedule deferred --steps 1 --warmup 3 2>/dev/null | grep -E "dram__|gpu__time" | awk -F'","' -v v=$v '{print v, $(NF-2), $NF}'
  fi
done
done
