# A/B: the pipelined (group-chunked, two-stream) schedule vs the two-call path, per workload and
# chunk size. Prints ms per step (device-timed) and the bench's unique-byte bandwidth.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_pipelined.py -q -x 2>&1 | tail -3
run() {  # workload schedule extra...
  timeout 300 python bench.py --workload $1 --schedule $2 "${@:3}" --steps 20 --warmup 5 --no-e2e --no-cpu-baseline \
    --no-variants 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); c=d['config']
print('%-11s %-10s gpc=%-4s graph=%-5s ms=%.4f  launches/step=%d' % (c['workload'], c['schedule'], c.get('groups_per_chunk','-'), c['cuda_graph'], d['ms_per_step'], d['gpu_launches']//d['steps']))"
}
for rep in 1 2; do
  for w in pythia redteam; do
    run $w two-call
    for g in 1 2 4 8; do run $w pipelined --pipe-groups $g; done
    run $w pipelined
    run $w two-call --cuda-graph
    run $w pipelined --cuda-graph
    run $w pipelined --cuda-graph --pipe-groups 2
  done
done
for w in rhomath qwen_shard toy; do
  run $w two-call
  run $w pipelined
  run $w pipelined --pipe-groups 2
done
