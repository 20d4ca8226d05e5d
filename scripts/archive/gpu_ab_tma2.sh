run() { w=$1; shift; env $E timeout 600 python bench.py --workload $w --steps 20 --warmup 5 --no-e2e --no-cpu-baseline "$@" 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels']; print('$E $w', round(d['ms_per_step'],4), 'fwd', round(k['fwd_ms'],4), round(k['fwd_gbs']))"; }
E=""; run qwen_shard
for c in 0 1 2 3; do E="TBA_FWD_IMPL=tma TBA_TMA_CFG=$c"; run qwen_shard; done
E=""; run qwen_shard
