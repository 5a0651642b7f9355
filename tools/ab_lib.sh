#!/bin/bash
# Interleaved A/B of library variants (tools/build_variant.sh) on one box:
#   VARIANTS="default epi_sleep" REPS=3 tools/ab_lib.sh
# prints per run: variant, ms/step, in-step GEMM ms, attribution ms per GEMM mode.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
for rep in $(seq ${REPS:-3}); do
  for v in ${VARIANTS:-default}; do
    if [ "$v" = default ]; then lib=""; else lib="$PWD/paper_2412_09952_b200/lib/variants/$v/libb200moe.so"; fi
    B200MOE_LIB=$lib python bench.py --steps ${STEPS:-30} --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/ab_$v.json 2> gpurun_out/ab_$v.err
    python -c "
import json;d=json.load(open('gpurun_out/ab_$v.json'))
k=d['kernels_ms_per_step']
print('$v', d['ms_per_step'], d['roofline']['gemm_ms_per_step'], d['clocks']['sm_mhz'], ' '.join(f'{n[7:]}={t}' for n,t in k.items() if n.startswith('expert')), '|', ' '.join(f'{n}={t}' for n,t in k.items() if not n.startswith('expert')))" || tail -3 gpurun_out/ab_$v.err
  done
done
