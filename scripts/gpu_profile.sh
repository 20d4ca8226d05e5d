# ncu evidence for profiles/: launch list (full shard), DRAM bytes per launch (full shard),
# and one --set full capture per hot kernel on a one-group slice. Usage: bash scripts/gpu_profile.sh TAG
set -x
TAG=${1:-r01}
mkdir -p gpurun_out
B="python bench.py --no-e2e --no-cpu-baseline --no-variants"
ncu --metrics gpu__time_duration.sum --clock-control none -s 12 -c 12 --csv --log-file gpurun_out/launches_${TAG}.csv $B --steps 4 --warmup 3 > gpurun_out/launches_bench_${TAG}.log 2>&1
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:row_ -s 6 -c 4 --csv --log-file gpurun_out/dram_${TAG}.csv $B --steps 2 --warmup 3 > /dev/null 2>&1
for K in row_bwd row_fwd_rows seq_head; do
  ncu --set full --clock-control none --import-source on -k regex:$K -s 3 -c 1 -o gpurun_out/prof_${K}_${TAG} -f $B --workload qwen_group --steps 1 --warmup 3 > gpurun_out/prof_${K}_${TAG}.log 2>&1
done
ls -la gpurun_out
