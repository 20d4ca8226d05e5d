# N=2 bench flow with the loss all-reduce fused into the head kernel (peer memory), 2 ranks on cuda:0
for c in nccl peer; do
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 \
  bench.py --gpus 2 --steps 5 --warmup 3 --workload pythia --no-e2e --dist-backend gloo --share-gpu --collective $c 2> gpurun_out/mr_peer_$c.err | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', d['n_gpus'], d['value'], d['ms_per_step'], d['loss'], d['config']['collective'])" || tail -5 gpurun_out/mr_peer_$c.err
done
timeout 600 python -m pytest tests/test_gpu_peer.py -q 2>&1 | tail -1
