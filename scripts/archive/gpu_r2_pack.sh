# A/B: the forward with the token state packed in one register and 32-bit indices (pack) vs the product
mkdir -p gpurun_out
TBA_LIBRARY=$PWD/ab_libs/pack/libtba.so timeout 900 python -m pytest -q -m gpu tests/test_gpu_parity.py tests/test_gpu_hostile.py tests/test_gpu_fused.py 2>&1 | tail -3
B="python bench.py --no-e2e --no-cpu-baseline --no-variants"
for rep in 1 2; do
for v in prod pack; do
  if [ $v = prod ]; then L=""; else L="$PWD/ab_libs/$v/libtba.so"; fi
  for wl in qwen_shard math_t5_shard rhomath pythia; do
  TBA_LIBRARY=$L $B --workload $wl > gpurun_out/e3_${v}_$wl.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/e3_${v}_$wl.json')); k=d['kernels']; print('$v', '$wl', round(d['ms_per_step'],4), 'fwd', round(k['fwd_ms'],4), round(k['fwd_frac'],3), 'step', round(k['step_frac'],3), d['clocks']['sm_mhz'])"
  done
done
done
