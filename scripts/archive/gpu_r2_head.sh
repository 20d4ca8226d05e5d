# HEAD check: every GPU test, smoke, the default bench line and the deferred lines.
mkdir -p gpurun_out
TBA_PARITY_OUT=gpurun_out/parity_head.json timeout 2400 python -m pytest tests -q -m gpu -x 2>&1 | tail -6
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/head_qwen_shard.json 2> gpurun_out/head_qwen_shard.err; tail -c 400 gpurun_out/head_qwen_shard.json
for wl in qwen_shard pythia redteam rhomath math_t5_shard; do
  timeout 600 python bench.py --workload $wl --schedule deferred --no-e2e --no-cpu-baseline --no-variants > gpurun_out/head_${wl}_deferred.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/head_${wl}_deferred.json')); print('deferred', '$wl', round(d['ms_per_step'],4), round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])"
done
