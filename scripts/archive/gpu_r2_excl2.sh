# A/B: token exclusion with one copy of the consume step (excl2) vs the uniform slow-copy branch (product)
# vs no exclusion (noexcl, inexact for confident tokens)
mkdir -p gpurun_out
python scripts/ab_variants.py excl2=TBA_AB_EXCL2 noexcl=TBA_AB_NO_EXCL > /dev/null 2>&1
TBA_LIBRARY=/tmp/tba_variants/excl2/libtba.so timeout 1200 python -m pytest -q -m gpu tests/test_gpu_parity.py tests/test_gpu_hostile.py tests/test_gpu_fused.py tests/test_gpu_variants.py 2>&1 | tail -1
B="python bench.py --no-e2e --no-cpu-baseline --no-variants"
for rep in 1 2; do
for v in prod excl2 noexcl; do
  if [ $v = prod ]; then L=""; else L="/tmp/tba_variants/$v/libtba.so"; fi
  for wl in qwen_shard rhomath pythia; do
  TBA_LIBRARY=$L $B --workload $wl > gpurun_out/ex_${v}_$wl.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/ex_${v}_$wl.json')); k=d['kernels']; print('$v', '$wl', round(d['ms_per_step'],4), 'fwd', round(k['fwd_ms'],4), round(k['fwd_frac'],3), 'bwd', round(k['bwd_ms'],4), 'step', round(k['step_frac'],3), d['clocks']['sm_mhz'])"
  done
done
done
