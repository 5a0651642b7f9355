#!/bin/bash
# Run the GPU test stages one process each (a faulting kernel poisons its
# CUDA context), each under its own timeout; logs land in gpurun_out/.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
nvidia-smi -L > gpurun_out/gpu.txt 2>&1
python -c "import numpy; numpy.show_runtime()" > gpurun_out/np_runtime.txt 2>&1
lscpu > gpurun_out/lscpu.txt 2>&1
status=0
for sel in "$@"; do
  name=$(echo "$sel" | tr -c 'A-Za-z0-9_' '_' | cut -c1-60)
  timeout ${STAGE_TIMEOUT:-600} python -m pytest $sel -q -m gpu -p no:cacheprovider > gpurun_out/t_$name.log 2>&1
  rc=$?
  echo "== $sel rc=$rc"; tail -25 gpurun_out/t_$name.log | cut -c1-400
  [ $rc -ne 0 ] && status=1
done
exit $status
