# seq_head with 8 loads in flight per lane: parity, head duration (ncu), forward ms on the small shapes.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_variants.py tests/test_gpu_tbap.py -q -x 2>&1 | tail -2
for w in qwen_shard pythia rhomath redteam gsm8k_k40; do
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:seq_head -c 3 --csv python bench.py --workload $w --no-e2e --no-cpu-baseline --no-variants --steps 2 --warmup 1 2>/dev/null | grep seq_head | awk -F'","' -v w=$w '{print w, $(NF)}' | tail -2
done
for w in pythia redteam gsm8k_t3 qwen_shard; do
  timeout 300 python bench.py --workload $w --no-e2e --no-cpu-baseline --no-variants --steps 30 --warmup 5 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels']; print('$w', round(d['ms_per_step'],4), round(k['fwd_ms'],4), round(k['fwd_gbs']))"
done
