#!/bin/bash
# Launch list (ncu, cold, serialised) of the non-GEMM b200moe kernels of the
# bench step, plus one normal bench run for the in-step event timings.
python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 > gpurun_out/small_bench_step.json
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none \
  -k 'regex:router|dispatch|permute|combine|reduce|importance|swizzle' --csv \
  --log-file gpurun_out/small_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
echo done
