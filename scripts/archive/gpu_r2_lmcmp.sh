# The one-call LM-head training step, round-2 build vs the round-1 library (build/r1), same box, interleaved.
mkdir -p gpurun_out
for rep in 1 2; do
for v in prod r1; do
  if [ $v = prod ]; then L=""; else L="$PWD/build/r1/libtba.so"; fi
  TBA_LIBRARY=$L timeout 900 python bench.py --workload qwen_shard --objective lmhead_train --steps 8 --warmup 3 --no-variants > gpurun_out/lmc_${v}.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/lmc_${v}.json').read().strip().splitlines()[-1]); print('$v', round(d['ms_per_step'],2), d['clocks']['sm_mhz'], d['kernels'])"
done
done
