#!/bin/bash
# A/B of backward GEMM schedules (B200MOE_BWD_SCHED, moe._bwd_schedule):
# interleaved bench runs on one box; prints ms_per_step and GEMM ms per variant.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
for rep in 1 2 3; do
  for sched in ${SCHEDS:-serial split:60 dag:96:60}; do
    B200MOE_BWD_SCHED=$sched python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/ab_$sched.json 2>/dev/null
    python -c "
import json,sys;d=json.load(open('gpurun_out/ab_$sched.json'))
print('$sched', d['ms_per_step'], d['roofline']['gemm_ms_per_step'], d['clocks']['sm_mhz'], {k:v for k,v in d['kernels_ms_per_step'].items() if 'expert' in k})"
  done
done
