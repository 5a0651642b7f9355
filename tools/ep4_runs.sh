cd ${GRAFT_REPO_ROOT:-/root/repo}
export PYTORCH_CUDA_ALLOC_CONF=expandable_segments:True
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 4 > gpurun_out/ep4.json 2>gpurun_out/ep4.err; echo ep4 rc=$?
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29512 tools/model_bench.py --layers 32 --experts 4 --micro-batches 8 --zero --recompute 16 --cf 1.0 --steps 3 --warmup 2 > gpurun_out/model32_cf1.log 2>&1; echo m1 rc=$?
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29513 tools/model_bench.py --layers 32 --experts 4 --micro-batches 8 --zero --recompute 32 --cf 2.0 --steps 3 --warmup 2 > gpurun_out/model32_cf2.log 2>&1; echo m2 rc=$?
