#!/bin/bash
# 32-layer EP4 (E=4, one expert per GPU) model step at reference CF 2 (the paper's CF 1): recompute / drop-h plans
cd ${GRAFT_REPO_ROOT:-$(dirname "$0")/..}
export PYTORCH_CUDA_ALLOC_CONF=expandable_segments:True
for RC in ${RCS:-16 12}; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29520+RC)) tools/model_bench.py --layers 32 --experts 4 --micro-batches ${MB:-8} --zero --recompute $RC --drop-h --cf 2.0 --steps 3 --warmup 2 > gpurun_out/model32_cf2_rc${RC}_droph_mb${MB:-8}.log 2>&1; echo rc$RC exit=$?
done
