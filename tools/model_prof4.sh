#!/bin/bash
# 32-layer EP4 model step at the paper's CF (reference CF 2) with a torch.profiler kernel breakdown per rank
cd ${GRAFT_REPO_ROOT:-$(dirname "$0")/..}
export PYTORCH_CUDA_ALLOC_CONF=expandable_segments:True
RC=${RC:-32}
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29514 tools/model_bench.py --layers 32 --experts 4 --micro-batches 8 --zero --recompute $RC ${EXTRA} --cf 2.0 --steps 2 --warmup 2 --profile > gpurun_out/model32_prof.log 2>&1; echo prof rc=$?
