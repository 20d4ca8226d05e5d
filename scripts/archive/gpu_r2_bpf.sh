# A/B: row_bwd with an L2 bulk prefetch 32 KB (bpf2) / 64 KB (bpf4) ahead of its loop vs none (the product)
mkdir -p gpurun_out
TBA_LIBRARY=$PWD/ab_libs/bpf4/libtba.so timeout 900 python -m pytest -q -m gpu tests/test_gpu_parity.py tests/test_gpu_guard.py 2>&1 | tail -1
B="python bench.py --no-e2e --no-cpu-baseline --no-variants"
for rep in 1 2; do
for v in prod bpf2 bpf4; do
  if [ $v = prod ]; then L=""; else L="$PWD/ab_libs/$v/libtba.so"; fi
  for wl in qwen_shard math_t5_shard rhomath pythia; do
  TBA_LIBRARY=$L $B --workload $wl > gpurun_out/bp_${v}_$wl.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/bp_${v}_$wl.json')); k=d['kernels']; print('$v', '$wl', round(d['ms_per_step'],4), 'fwd', round(k['fwd_ms'],4), 'bwd', round(k['bwd_ms'],4), round(d['roofline']['frac'],3), 'step', round(k['step_frac'],3), d['clocks']['sm_mhz'])"
  done
done
done
