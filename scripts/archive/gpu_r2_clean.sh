# After removing the unused cluster / REV / stash paths of bwd_row and the deferred kernel: every GPU
# test, and bench lines against the previous HEAD's library (headref, built from a git worktree copy)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -x 2>&1 | tail -3
B="python bench.py --no-e2e --no-cpu-baseline --no-variants"
for rep in 1 2; do
for v in prod headref; do
  if [ $v = prod ]; then L=""; else L="$PWD/gpurun_out/headref/libtba.so"; fi
  for wl in qwen_shard pythia rhomath; do
  TBA_LIBRARY=$L $B --workload $wl > gpurun_out/cl_${v}_$wl.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/cl_${v}_$wl.json')); k=d['kernels']; print('$v', '$wl', round(d['ms_per_step'],4), 'fwd', round(k['fwd_ms'],4), 'bwd', round(k['bwd_ms'],4), 'step', round(k['step_frac'],3), d['clocks']['sm_mhz'])"
  TBA_LIBRARY=$L $B --workload $wl --schedule deferred > gpurun_out/cl_${v}_${wl}_d.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/cl_${v}_${wl}_d.json')); print('$v', '$wl', 'deferred', round(d['ms_per_step'],4), round(d['roofline']['frac'],3))"
  done
done
done
