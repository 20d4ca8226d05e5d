# A/B on the large-group shapes: pipelined with few chunks vs two-call, interleaved.
run() {
  timeout 300 python bench.py --workload $1 --schedule $2 "${@:3}" --steps 30 --warmup 5 --no-e2e --no-cpu-baseline \
    --no-variants 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); c=d['config']
print('%-11s %-10s gpc=%-4s ms=%.4f' % (c['workload'], c['schedule'], c.get('groups_per_chunk','-'), d['ms_per_step']))"
}
for rep in 1 2 3; do
  run qwen_shard two-call
  for g in 1 2 3 4; do run qwen_shard pipelined --pipe-groups $g; done
done
for rep in 1 2; do
  run rhomath two-call
  for g in 4 8 16; do run rhomath pipelined --pipe-groups $g; done
done
