# Same box, interleaved: the round-1 library (commit 7c5e1fe, ab_libs/r1) vs the final round-2 build
mkdir -p gpurun_out
B="python bench.py --no-e2e --no-cpu-baseline --no-variants"
for rep in 1 2 3; do
for v in prod r1; do
  if [ $v = prod ]; then L=""; else L="$PWD/ab_libs/$v/libtba.so"; fi
  for wl in qwen_shard rhomath pythia redteam; do
  TBA_LIBRARY=$L $B --workload $wl > gpurun_out/rc_${v}_$wl.json 2>gpurun_out/rc_${v}_$wl.err
  python -c "
import json; d=json.load(open('gpurun_out/rc_${v}_$wl.json')); k=d['kernels']; print('$v', '$wl', round(d['ms_per_step'],4), 'fwd', round(k['fwd_ms'],4), 'bwd', round(k['bwd_ms'],4), 'step', round(k['step_frac'],3), d['clocks']['sm_mhz'])" 2>/dev/null || echo "$v $wl failed: $(tail -1 gpurun_out/rc_${v}_$wl.err)"
  done
  TBA_LIBRARY=$L $B --workload qwen_shard --schedule deferred > gpurun_out/rc_${v}_qd.json 2>gpurun_out/rc_${v}_qd.err
  python -c "
import json; d=json.load(open('gpurun_out/rc_${v}_qd.json')); print('$v', 'qwen deferred', round(d['ms_per_step'],4), round(d['roofline']['frac'],3))" 2>/dev/null || echo "$v deferred failed: $(tail -1 gpurun_out/rc_${v}_qd.err)"
done
done
