# NEXT 2 (i) with PDL: the group-chunk schedule on one stream (chunk kernels PDL-chained, the writer
# of chunk c re-reading it from L2 right after its forward) vs two streams vs the two-call step.
mkdir -p gpurun_out
for wl in pythia redteam tldr_t4 gsm8k_t3; do
  timeout 300 python bench.py --workload $wl --no-e2e --no-cpu-baseline --no-variants > gpurun_out/pp_two_$wl.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/pp_two_$wl.json')); print('$wl two-call', round(d['ms_per_step'],4))"
  for g in 1 2 4 8; do
    for mode in "" "--pipe-one-stream"; do
      timeout 300 python bench.py --workload $wl --schedule pipelined --pipe-groups $g $mode --no-e2e --no-cpu-baseline --no-variants > gpurun_out/pp.json 2>/dev/null
      python -c "import json; d=json.load(open('gpurun_out/pp.json')); print('$wl pipelined g=$g $mode', round(d['ms_per_step'],4))"
    done
  done
  timeout 300 python bench.py --workload $wl --schedule fused --no-e2e --no-cpu-baseline --no-variants > gpurun_out/pp.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/pp.json')); print('$wl fused', round(d['ms_per_step'],4))"
done
