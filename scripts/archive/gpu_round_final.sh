# Round-end evidence: tests, smoke, profiles, bench lines for every workload, sanitizers.
TAG=${1:-r01}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
bash scripts/gpu_profile.sh $TAG > /dev/null 2>&1
bash scripts/gpu_bench_all.sh $TAG
timeout 600 python bench.py --objective tbap --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_${TAG}_qwen_shard_tbap.json 2>/dev/null
tail -c 600 gpurun_out/bench_${TAG}_qwen_shard_tbap.json
bash scripts/gpu_sanitize.sh
for w in qwen_shard rhomath pythia redteam; do timeout 600 python bench.py --workload $w --schedule deferred --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/bench_${TAG}_${w}_deferred.json 2>/dev/null; done
bash scripts/gpu_lmhead.sh $TAG > /dev/null 2>&1
tail -c 300 gpurun_out/bench_${TAG}_qwen_shard_lmhead.json
timeout 600 python bench.py --workload toy --cuda-graph --steps 50 --warmup 10 --no-e2e --no-cpu-baseline > gpurun_out/bench_${TAG}_toy_graph.json 2>/dev/null
# LM-head forward + backward (NEXT 3): bench lines (one-call vs two-call vs cuBLAS) and the launch list
bash scripts/gpu_lmtrain.sh $TAG
timeout 600 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg.per_second,lts__t_sector_hit_rate.pct,lts__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none --csv --log-file gpurun_out/lmtrain_launches_${TAG}.csv python scripts/lm_bwd_probe.py --one-call > /dev/null 2>&1
