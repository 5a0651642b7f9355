#!/bin/bash
# Multi-GPU evidence on one 4-GPU box: EP2 and EP4 bench lines, then the 32-layer model step at the paper's CF
# (reference CF 2: drop-h + recompute in 16 layers) and at reference CF 1 (recompute in 16 layers).
cd ${GRAFT_REPO_ROOT:-$(dirname "$0")/..}
export PYTORCH_CUDA_ALLOC_CONF=expandable_segments:True
mkdir -p gpurun_out/ev
for N in 2 4; do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29700+N)) bench.py --gpus $N > gpurun_out/ev/bench_ep$N.json 2> gpurun_out/ev/bench_ep$N.err; echo ep$N rc=$?
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29711 tools/model_bench.py --layers 32 --experts 4 --micro-batches 8 --zero --recompute 16 --drop-h --cf 2.0 --steps 3 --warmup 2 > gpurun_out/ev/model_cf2.log 2>&1; echo m2 rc=$?
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29712 tools/model_bench.py --layers 32 --experts 4 --micro-batches 8 --zero --recompute 16 --cf 1.0 --steps 3 --warmup 2 > gpurun_out/ev/model_cf1.log 2>&1; echo m1 rc=$?
