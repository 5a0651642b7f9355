#!/bin/bash
# A/B of a BWD2 variant: A = the built library, B = gemm.cu rebuilt with $AB_FLAGS (e.g. -DB200_BWD2_LOAD_BUFS=2 -DB200_BWD2_CHUNK16=0)
cd ${GRAFT_REPO_ROOT:-.}
L=paper_2412_09952_b200/lib
cp $L/libb200moe.so $L/libb200moe_a.so
cd paper_2412_09952_b200/csrc
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -ftz=false -prec-div=true -prec-sqrt=true $AB_FLAGS -c gemm.cu -o /tmp/gemm_b.o
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o ../lib/libb200moe_b.so ../lib/obj/capi.o ../lib/obj/router.o ../lib/obj/permute.o ../lib/obj/router_bwd.o /tmp/gemm_b.o ../lib/obj/upcycle.o ../lib/obj/model.o ../lib/obj/crc32c.o
cd ../..
for r in 1 2 3 4; do for v in a b; do
  cp $L/libb200moe_$v.so $L/libb200moe.so
  timeout 200 python bench.py --steps 40 --warmup 5 --no-cpu-baseline --no-e2e | python -c "import json,sys; l=json.loads(sys.stdin.read()); k=l['kernels_ms_per_step']; print('$v', l['ms_per_step'], k['expert_bwd2'], k['expert_fwd2'])"
done; done
cp $L/libb200moe_a.so $L/libb200moe.so
