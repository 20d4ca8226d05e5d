# Round-2 check at HEAD: every GPU test (parity maxima -> gpurun_out/parity_r02.json), smoke, the default
# bench line, the N>1 flow (2 ranks sharing cuda:0 over gloo; weak and strong), strong scaling at N=1,
# the reference arm.
mkdir -p gpurun_out
echo "cores: $(nproc)"
TBA_PARITY_OUT=gpurun_out/parity_r02.json timeout 2400 python -m pytest tests -q -m gpu --durations=15 2>&1 | tail -25
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err; tail -c 2500 gpurun_out/r2_bench.json
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 \
  bench.py --gpus 2 --steps 5 --warmup 3 --workload pythia --dist-backend gloo --share-gpu --no-variants 2>&1 | grep -v Warning | tail -2 | cut -c1-600
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 \
  bench.py --gpus 2 --steps 3 --warmup 3 --workload rhomath --scaling strong --chunk-groups 4 --dist-backend gloo --share-gpu 2>&1 | grep -v Warning | tail -2 | cut -c1-900
timeout 900 python bench.py --scaling strong --workload qwen --steps 5 --warmup 3 > gpurun_out/r2_strong_qwen.json 2>&1; tail -c 1500 gpurun_out/r2_strong_qwen.json
timeout 900 python bench.py --impl reference > gpurun_out/r2_ref.json 2>&1; tail -c 1500 gpurun_out/r2_ref.json
