# Exercise bench.py's N>1 flow on ONE GPU: 2 ranks share cuda:0 over gloo (NCCL rejects duplicate GPUs).
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 \
  bench.py --gpus 2 --steps 5 --warmup 3 --workload pythia --dist-backend gloo --share-gpu 2>&1 | grep -v Warning | tail -3
