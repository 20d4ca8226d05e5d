# The LM-head-fused forward (objective lmhead), round-2 build vs the round-1 library, same box, interleaved.
mkdir -p gpurun_out
for rep in 1 2 3; do
for v in prod r1; do
  if [ $v = prod ]; then L=""; else L="$PWD/build/r1/libtba.so"; fi
  TBA_LIBRARY=$L timeout 900 python bench.py --workload qwen_shard --objective lmhead --steps 10 --warmup 3 --no-variants --no-e2e --no-cpu-baseline > gpurun_out/lmf_${v}.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/lmf_${v}.json').read().strip().splitlines()[-1]); print('$v', round(d['ms_per_step'],2), d['clocks']['sm_mhz'])"
done
done
