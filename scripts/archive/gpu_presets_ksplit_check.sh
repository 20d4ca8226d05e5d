mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_lmhead_bwd.py -x -q 2>&1 | tail -2
bash scripts/gpu_sanitize.sh 2>&1 | tail -14
for w in math_t5_shard gsm8k_t3 tldr_t4 gsm8k_k40; do timeout 600 python bench.py --workload $w --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/bench_r01_$w.json 2>gpurun_out/bench_r01_$w.err; python -c "
import json,sys; d=json.load(open('gpurun_out/bench_r01_$w.json')); print('$w', d['ms_per_step'], d['value'], d['roofline']['frac'], d['kernels'])"; done
