# A/B: forward tail split — the last N rows in a second PDL-chained grid with more threads per row
# (t2k: 2048 rows at 128 threads, t4k: 4096, t2k64: 2048 at 64) vs one grid (the product)
mkdir -p gpurun_out
TBA_LIBRARY=$PWD/ab_libs/t2k/libtba.so timeout 1200 python -m pytest -q -m gpu tests/test_gpu_parity.py tests/test_gpu_hostile.py tests/test_gpu_guard.py tests/test_gpu_fullsize.py -k "not fused and not pipelined" 2>&1 | tail -2
B="python bench.py --no-e2e --no-cpu-baseline --no-variants"
for rep in 1 2; do
for v in prod t2k t4k t2k64; do
  if [ $v = prod ]; then L=""; else L="$PWD/ab_libs/$v/libtba.so"; fi
  for wl in pythia redteam gsm8k_t3 gsm8k_k40 rhomath tldr_t4; do
  TBA_LIBRARY=$L $B --workload $wl > gpurun_out/tl_${v}_$wl.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/tl_${v}_$wl.json')); k=d['kernels']; print('$v', '$wl', round(d['ms_per_step'],4), 'fwd', round(k['fwd_ms'],4), round(k['fwd_frac'],3), 'bwd', round(k['bwd_ms'],4), 'step', round(k['step_frac'],3), d['clocks']['sm_mhz'])"
  done
done
done
