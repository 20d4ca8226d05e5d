# A/B: the forward requests a row's mask and token together (product candidate), + the token-dependent
# setup after the first loads (lazy) vs the previous HEAD (headref)
mkdir -p gpurun_out
timeout 900 python -m pytest -q -m gpu tests/test_gpu_parity.py tests/test_gpu_hostile.py tests/test_gpu_guard.py tests/test_gpu_variants.py 2>&1 | tail -1
TBA_LIBRARY=$PWD/ab_libs/lazy/libtba.so timeout 900 python -m pytest -q -m gpu tests/test_gpu_parity.py tests/test_gpu_hostile.py 2>&1 | tail -1
B="python bench.py --no-e2e --no-cpu-baseline --no-variants"
for rep in 1 2; do
for v in prod lazy headref; do
  if [ $v = prod ]; then L=""; else L="$PWD/ab_libs/$v/libtba.so"; fi
  for wl in pythia redteam gsm8k_t3 rhomath qwen_shard; do
  TBA_LIBRARY=$L $B --workload $wl > gpurun_out/ea_${v}_$wl.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/ea_${v}_$wl.json')); k=d['kernels']; print('$v', '$wl', round(d['ms_per_step'],4), 'fwd', round(k['fwd_ms'],4), round(k['fwd_frac'],3), 'step', round(k['step_frac'],3), d['clocks']['sm_mhz'])"
  done
done
done
