# A/B of forward implementations. Usage: bash scripts/gpu_ab.sh [cfgs...]
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
run() { env "$@" timeout 600 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels']; print('$*', round(d['ms_per_step'],3), 'fwd', round(k['fwd_ms'],3), round(k['fwd_gbs']), 'bwd', round(k['bwd_ms'],3), round(k['bwd_gbs']), d['clocks']['sm_mhz'], d['clocks']['reasons'])"; }
run TBA_FWD_IMPL=ldg
for c in ${@:-0 1 2 3 4 5}; do run TBA_FWD_IMPL=tma TBA_TMA_CFG=$c; done
