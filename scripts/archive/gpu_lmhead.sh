# NEXT 3 evidence: bench line (objective lmhead), launch list, DRAM bytes and one ncu --set full
# capture of lmhead_fwd on the Qwen shard. Usage: bash scripts/gpu_lmhead.sh TAG
TAG=${1:-r01}
mkdir -p gpurun_out
timeout 900 python bench.py --objective lmhead --steps 10 --warmup 3 > gpurun_out/bench_${TAG}_qwen_shard_lmhead.json 2> gpurun_out/bench_${TAG}_lmhead.err
tail -c 2500 gpurun_out/bench_${TAG}_qwen_shard_lmhead.json
timeout 900 python bench.py --objective lmhead --workload rhomath --steps 10 --warmup 3 > gpurun_out/bench_${TAG}_rhomath_lmhead.json 2>/dev/null
B="python bench.py --objective lmhead --no-e2e --no-cpu-baseline --no-variants"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 9 -c 6 --csv --log-file gpurun_out/lmhead_launches_${TAG}.csv $B --steps 2 --warmup 3 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:lmhead_fwd -s 3 -c 1 -o gpurun_out/prof_lmhead_fwd_${TAG} -f $B --steps 1 --warmup 3 > gpurun_out/prof_lmhead_fwd_${TAG}.log 2>&1
tail -3 gpurun_out/prof_lmhead_fwd_${TAG}.log
