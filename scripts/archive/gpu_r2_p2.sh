# A/B: the deferred pass 2 without per-vector bounds/stash tests (product candidate) vs bwd_row's loop (oldp2)
mkdir -p gpurun_out
python scripts/ab_variants.py oldp2=TBA_AB_OLD_P2 > /dev/null 2>&1
timeout 900 python -m pytest -q -m gpu tests/test_gpu_fused.py tests/test_gpu_tbap.py tests/test_gpu_hostile.py -k "deferred or confident" 2>&1 | tail -1
for rep in 1 2; do
for v in prod oldp2; do
  if [ $v = prod ]; then L=""; else L="/tmp/tba_variants/$v/libtba.so"; fi
  for wl in qwen_shard math_t5_shard pythia_fp32; do
    TBA_LIBRARY=$L timeout 300 python bench.py --workload $wl --schedule deferred --no-e2e --no-cpu-baseline --no-variants > gpurun_out/p2_${v}_$wl.json 2>gpurun_out/p2_${v}_$wl.err
    python -c "
import json; d=json.load(open('gpurun_out/p2_${v}_$wl.json')); print('$v', '$wl', round(d['ms_per_step'],4), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])" || tail -3 gpurun_out/p2_${v}_$wl.err
  done
  TBA_LIBRARY=$L python scripts/microbench/defer_steps.py 2>&1 | python -c "
import sys
for l in sys.stdin:
    if 'sleep' in l:
        p=l.split(); t=sorted(map(float,p[3:])); print('$v', p[0], p[1], p[2], 'median', t[len(t)//2], 'min', t[0])
"
done
done
ncu --set full --clock-control none --import-source on -k regex:row_single -s 3 -c 1 -o gpurun_out/prof_row_single_p2 -f python bench.py --no-e2e --no-cpu-baseline --no-variants --workload qwen_group --schedule deferred --steps 1 --warmup 3 > /dev/null 2>&1
