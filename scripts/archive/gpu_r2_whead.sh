# Warp-parallel group head (product candidate) vs the previous HEAD (ab_libs/headref): every GPU test,
# the presets with K = 20 / 40 and the Qwen shard
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -x 2>&1 | tail -3
B="python bench.py --no-e2e --no-cpu-baseline --no-variants"
for rep in 1 2; do
for v in prod headref; do
  if [ $v = prod ]; then L=""; else L="$PWD/ab_libs/$v/libtba.so"; fi
  for wl in gsm8k_k40 gsm8k_t3 tldr_t4 rhomath pythia qwen_shard; do
  TBA_LIBRARY=$L $B --workload $wl > gpurun_out/wh_${v}_$wl.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/wh_${v}_$wl.json')); k=d['kernels']; print('$v', '$wl', round(d['ms_per_step'],4), 'fwd', round(k['fwd_ms'],4), round(k['fwd_frac'],3), 'bwd', round(k['bwd_ms'],4), 'step', round(k['step_frac'],3), d['clocks']['sm_mhz'])"
  done
done
done
for v in prod headref; do
  if [ $v = prod ]; then L=""; else L="$PWD/ab_libs/$v/libtba.so"; fi
  TBA_LIBRARY=$L ncu --metrics gpu__time_duration.sum --clock-control none -k regex:seq_head -s 3 -c 2 --csv $B --workload gsm8k_k40 --steps 2 --warmup 3 2>/dev/null | grep gpu__time | awk -F'","' -v v=$v '{print v, "seq_head k40 ns", $NF}'
  TBA_LIBRARY=$L ncu --metrics gpu__time_duration.sum --clock-control none -k regex:seq_head -s 3 -c 2 --csv $B --workload pythia --steps 2 --warmup 3 2>/dev/null | grep gpu__time | awk -F'","' -v v=$v '{print v, "seq_head pythia ns", $NF}'
done
