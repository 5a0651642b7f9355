#!/bin/bash
# Config-4 ablation at the Llama-3 shape (single GPU): CF 1/2/4 x {mixtral, st}
# with the position policy, plus the score policy at CF 1 and 2 (and dropless).
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
for cf in 1.0 2.0 4.0; do
  for r in mixtral st; do
    timeout 300 python bench.py --steps 15 --warmup 4 --cf $cf --router $r --no-cpu-baseline --no-e2e 2>/dev/null | grep "^{"
  done
  timeout 300 python bench.py --steps 15 --warmup 4 --cf $cf --router mixtral --policy score --no-cpu-baseline --no-e2e 2>/dev/null | grep "^{"
done
for r in mixtral st; do   # dropless (CF=None)
  timeout 300 python bench.py --steps 15 --warmup 4 --cf none --router $r --no-cpu-baseline --no-e2e 2>/dev/null | grep "^{"
done
