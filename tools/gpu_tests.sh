#!/bin/bash
# Run GPU test stages one process each (a faulting kernel poisons its CUDA
# context), each under its own timeout; logs land in gpurun_out/.
# Stage syntax: "path/to/test.py" or "path/to/test.py|<pytest -k expression>".
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
nvidia-smi -L > gpurun_out/gpu.txt 2>&1
python -c "import numpy; numpy.show_runtime()" > gpurun_out/np_runtime.txt 2>&1
lscpu > gpurun_out/lscpu.txt 2>&1
status=0
i=0
for sel in "$@"; do
  i=$((i+1))
  file="${sel%%|*}"
  if [[ "$sel" == *"|"* ]]; then kexpr="${sel#*|}"; else kexpr=""; fi
  log=gpurun_out/t_stage$i.log
  if [ -n "$kexpr" ]; then
    timeout ${STAGE_TIMEOUT:-600} python -m pytest "$file" -k "$kexpr" -q -m gpu -p no:cacheprovider > $log 2>&1
  else
    timeout ${STAGE_TIMEOUT:-600} python -m pytest "$file" -q -m gpu -p no:cacheprovider > $log 2>&1
  fi
  rc=$?
  echo "== stage $i: $sel rc=$rc"; tail -${TAIL:-25} $log | cut -c1-400
  [ $rc -ne 0 ] && status=1
done
exit $status
