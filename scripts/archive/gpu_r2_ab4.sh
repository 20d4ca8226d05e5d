# A/B 4: the product vs two loops around the token's iteration vs the round-1 library (build/r1,
# commit 7c5e1fe, built in a worktree); forward time on the Qwen shard and Pythia, interleaved, 3 repeats.
mkdir -p gpurun_out
python scripts/ab_variants.py noexcl=TBA_AB_NO_EXCL splitloop=TBA_AB_SPLIT_LOOP > /dev/null 2>&1
for rep in 1 2 3; do
for v in prod splitloop r1; do
  if [ $v = prod ]; then L=""; elif [ $v = r1 ]; then L="$PWD/build/r1/libtba.so"; else L="/tmp/tba_variants/$v/libtba.so"; fi
  for wl in qwen_shard pythia; do
    TBA_LIBRARY=$L timeout 600 python bench.py --workload $wl --no-e2e --no-cpu-baseline --no-variants > gpurun_out/ab4_${v}_$wl.json 2>/dev/null
    python -c "
import json; d=json.load(open('gpurun_out/ab4_${v}_$wl.json')); k=d['kernels']
print('$v', '$wl', round(d['ms_per_step'],4), 'fwd', round(k['fwd_ms'],4), 'bwd', round(k['bwd_ms'],4), d['clocks']['sm_mhz'])"
  done
done
done
