#!/bin/bash
# Same-box A/B of the EP return exchange: pushed from the FWD2 / BWD1 epilogues (default) vs pulled by combine /
# router backward (--ep-pull), N GPUs, interleaved.
cd ${GRAFT_REPO_ROOT:-$(dirname "$0")/..}
N=${N:-2}
for r in 1 2 3; do for v in push pull; do
  flag=""; [ $v = pull ] && flag="--ep-pull"
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29600+r*2+${#v})) bench.py --gpus $N --no-cpu-baseline $flag > gpurun_out/ab_ep_$v.json 2>/dev/null
  python -c "
import json; d=json.loads([l for l in open('gpurun_out/ab_ep_$v.json') if l.startswith('{')][-1])
print('$v', d['value'], d['ms_per_step'], d['roofline']['gemm_share_of_step'], {k: v for k, v in d['kernels_ms_per_step'].items() if 'fwd2' in k or 'bwd1' in k or 'combine_peer' in k or 'router_bwd' in k})"
done; done
