# A/B: per-sequence sums with 16 positions per lane in flight (product candidate) vs 8 (sb8); bitwise equal
mkdir -p gpurun_out
timeout 900 python -m pytest -q -m gpu tests/test_gpu_parity.py tests/test_gpu_fused.py tests/test_gpu_pipelined.py 2>&1 | tail -1
B="python bench.py --no-e2e --no-cpu-baseline --no-variants"
for rep in 1 2; do
for v in prod sb8; do
  if [ $v = prod ]; then L=""; else L="$PWD/ab_libs/$v/libtba.so"; fi
  for wl in gsm8k_k40 gsm8k_t3 tldr_t4 pythia qwen_shard; do
  TBA_LIBRARY=$L $B --workload $wl > gpurun_out/sb_${v}_$wl.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/sb_${v}_$wl.json')); k=d['kernels']; print('$v', '$wl', round(d['ms_per_step'],4), 'fwd', round(k['fwd_ms'],4), round(k['fwd_frac'],3), 'step', round(k['step_frac'],3), d['clocks']['sm_mhz'])"
  done
done
done
