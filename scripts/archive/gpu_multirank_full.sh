# bench.py's N=2 flow at the full Qwen shard (2 ranks share cuda:0 over gloo), e2e on; default runs timed.
t0=$(date +%s)
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 \
  bench.py --gpus 2 --steps 5 --warmup 3 --dist-backend gloo --share-gpu 2> gpurun_out/mr_full.err | tail -1 > gpurun_out/mr_full.json
echo "N=2 shared-GPU run: $(( $(date +%s) - t0 )) s"; python -c "import json; d=json.load(open('gpurun_out/mr_full.json')); print(d['n_gpus'], d['value'], d['ms_per_step'], d['e2e'], d['cpu_baseline'])" || tail -20 gpurun_out/mr_full.err
t0=$(date +%s); python bench.py > gpurun_out/default_bench.json 2> gpurun_out/default_bench.err; echo "default bench: $(( $(date +%s) - t0 )) s"; tail -c 400 gpurun_out/default_bench.json
t0=$(date +%s); python bench.py --impl reference > gpurun_out/default_ref.json 2> gpurun_out/default_ref.err; echo "reference arm: $(( $(date +%s) - t0 )) s"; cat gpurun_out/default_ref.json
