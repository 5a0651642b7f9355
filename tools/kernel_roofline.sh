#!/bin/bash
# ncu per-launch duration + DRAM bytes of the layer's memory-bound kernels (bench step)
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k 'regex:router|dispatch|permute|combine|reduce_partials|importance' --csv \
  --log-file gpurun_out/kernel_roofline.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
echo done
