timeout 900 python -m pytest tests/test_gpu_fused.py -q -k graph 2>&1 | tail -1
run() { w=$1; shift; timeout 600 python bench.py --workload $w --steps 50 --warmup 10 --no-e2e --no-cpu-baseline "$@" 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w $*', round(d['ms_per_step'],4), 'tok/s %.4g' % d['value'])"; }
for w in toy pythia redteam qwen_shard; do run $w; run $w --cuda-graph; done
