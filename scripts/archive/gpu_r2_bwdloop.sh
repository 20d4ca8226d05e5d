# A/B: row_bwd's vector loop without per-vector bounds tests (product candidate) vs the round-2 loop (oldbwd)
mkdir -p gpurun_out
python scripts/ab_variants.py oldbwd=TBA_AB_OLD_BWD > /dev/null 2>&1
timeout 1200 python -m pytest -q -m gpu tests/test_gpu_parity.py tests/test_gpu_fused.py tests/test_gpu_hostile.py tests/test_gpu_tbap.py tests/test_gpu_pipelined.py 2>&1 | tail -1
B="python bench.py --no-e2e --no-cpu-baseline --no-variants"
for rep in 1 2; do
for v in prod oldbwd; do
  if [ $v = prod ]; then L=""; else L="/tmp/tba_variants/$v/libtba.so"; fi
  for wl in qwen_shard pythia redteam rhomath; do
  TBA_LIBRARY=$L $B --workload $wl > gpurun_out/bl_${v}_$wl.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/bl_${v}_$wl.json')); k=d['kernels']; print('$v', '$wl', round(d['ms_per_step'],4), 'fwd', round(k['fwd_ms'],4), round(k['fwd_frac'],3), 'bwd', round(k['bwd_ms'],4), round(k.get('bwd_frac',0),3), 'step', round(k['step_frac'],3), d['clocks']['sm_mhz'])"
  done
done
done
