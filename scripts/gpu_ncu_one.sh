# One ncu --set full capture of a kernel on the one-group Qwen slice. Usage: bash scripts/gpu_ncu_one.sh REGEX TAG [env...]
K=$1; TAG=$2; shift 2
mkdir -p gpurun_out
env "$@" ncu --set full --clock-control none --import-source on -k regex:$K -s 3 -c 1 -o gpurun_out/prof_${TAG} -f python bench.py --no-e2e --no-cpu-baseline --workload qwen_group --steps 1 --warmup 3 > gpurun_out/prof_${TAG}.log 2>&1
tail -2 gpurun_out/prof_${TAG}.log
