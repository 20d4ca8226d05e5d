timeout 900 python -m pytest tests/test_gpu_fused.py -x -q -k "deferred" 2>&1 | tail -1
run() { w=$1; shift; env $E timeout 600 python bench.py --workload $w --steps 20 --warmup 5 --no-e2e --no-cpu-baseline "$@" 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$E $w $*', round(d['ms_per_step'],4), 'tok/s %.4g' % d['value'], 'roof %.0f %.3f' % (r['achieved'], r['frac']))"; }
for c in 2 3 4 5 6; do E="TBA_SINGLE_CFG=$c"; run qwen_shard --schedule deferred; done
