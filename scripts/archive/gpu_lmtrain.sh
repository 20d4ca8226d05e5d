# LM-head fused forward + backward (NEXT 3): bench lines on Qwen and RhoMath shards.
TAG=${1:-r01}
mkdir -p gpurun_out
timeout 900 python bench.py --objective lmhead_train --steps 4 --warmup 3 > gpurun_out/bench_${TAG}_qwen_shard_lmtrain.json 2> gpurun_out/lmtrain.err
tail -c 1500 gpurun_out/bench_${TAG}_qwen_shard_lmtrain.json; tail -5 gpurun_out/lmtrain.err
timeout 600 python bench.py --objective lmhead_train --workload rhomath --steps 4 --warmup 3 > gpurun_out/bench_${TAG}_rhomath_lmtrain.json 2>> gpurun_out/lmtrain.err
tail -c 1200 gpurun_out/bench_${TAG}_rhomath_lmtrain.json
