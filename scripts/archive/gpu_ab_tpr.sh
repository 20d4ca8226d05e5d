run() { w=$1; shift; env "$@" timeout 600 python bench.py --workload $w --steps 30 --warmup 5 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels']; print('$w $*', round(d['ms_per_step'],4), 'fwd', round(k['fwd_ms'],4), round(k['fwd_gbs']), 'bwd', round(k['bwd_ms'],4), round(k['bwd_gbs']))"; }
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
for w in pythia rhomath redteam qwen_shard; do for t in 0 32 64 128 256; do run $w TBA_FWD_TPR=$t; done; done
