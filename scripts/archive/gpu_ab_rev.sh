# Deferred pass: pass-2 sweep reversed (cfg 8 = cfg 4 reversed, cfg 9 = cfg 0 reversed).
TBA_SINGLE_CFG=8 timeout 300 python -m pytest tests/test_gpu_fused.py -q -x -k deferred 2>&1 | tail -1
TBA_SINGLE_CFG=9 timeout 300 python -m pytest tests/test_gpu_fused.py -q -x -k deferred 2>&1 | tail -1
run() {
  env "$@" timeout 300 python bench.py --workload $W --schedule deferred --steps 20 --warmup 5 --no-e2e --no-cpu-baseline \
    --no-variants 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('%-12s %-20s ms=%.4f' % ('$W', '$*', d['ms_per_step']))"
}
for rep in 1 2; do
  W=qwen_shard; run TBA_SINGLE_CFG=4; run TBA_SINGLE_CFG=8
  W=rhomath; run TBA_SINGLE_CFG=0; run TBA_SINGLE_CFG=9
  W=pythia; run TBA_SINGLE_CFG=0; run TBA_SINGLE_CFG=9
done
B="python bench.py --schedule deferred --no-e2e --no-cpu-baseline --no-variants --steps 1 --warmup 3"
for c in 4 8; do TBA_SINGLE_CFG=$c timeout 300 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum --clock-control none -k regex:row_single -s 3 -c 1 --csv $B 2>/dev/null | grep -E "dram__bytes_read|duration" | awk -F'","' -v t="cfg=$c" '{print t, $(NF-2), $NF}'; done
