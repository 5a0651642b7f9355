#!/bin/bash
# Round-2 evidence on one B200 (each ncu pass after the same command exited 0
# without ncu): the bench line (driver defaults), the reference arm, the ncu
# launch list of a bench run, one ncu --set full capture of a whole step's
# kernels, the config-4 ablation and the dense-projection A/B.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
OUT=gpurun_out/r02
mkdir -p $OUT
python bench.py --steps 20 --warmup 5 > $OUT/bench.json 2> $OUT/bench.err || { tail $OUT/bench.err; exit 1; }
python bench.py --impl reference --steps 3 --warmup 1 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
  --log-file $OUT/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/plain1.log 2>&1 && \
timeout 1200 ncu --set full --import-source on --clock-control none \
  --metrics sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_tc.sum \
  -k regex:"moe_gemm_kernel|router_|dispatch_scan|permute_kernel|combine|importance_bwd" -s 42 -c 14 \
  -o $OUT/step_full python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $OUT/ncu_full.log 2>&1
bash tools/ablation.sh > $OUT/ablation.jsonl 2> /dev/null
python tools/dense_bench.py > $OUT/dense_bench.json 2> /dev/null
python tools/router_ab.py > $OUT/router_ab.txt 2> /dev/null
ls -la $OUT
