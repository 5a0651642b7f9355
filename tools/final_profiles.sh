#!/bin/bash
# Round evidence on one B200: the bench line, its ncu launch list, one full ncu
# capture of a step's five grouped-GEMM launches (DRAM traffic for
# roofline.traffic), the model-step bench and the microbenchmarks.  Every ncu
# pass runs after the same command has exited 0 without ncu.
set -u
OUT=gpurun_out/final
mkdir -p $OUT
python bench.py --steps 30 --warmup 5 > $OUT/bench.json 2> $OUT/bench.err || exit 1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
  --log-file $OUT/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:moe_gemm -s 15 -c 5 \
  -o $OUT/gemm_step python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 600 python tools/model_bench.py --layers 2 > $OUT/model_1gpu.json 2> $OUT/model.err
python tools/gemm_bench.py > $OUT/gemm_bench.json 2>/dev/null
python tools/small_bench.py > $OUT/small_bench.json 2>/dev/null
python tools/opt_bench.py --gparams 2 > $OUT/opt_bench.json 2>/dev/null
python tools/crc_bench.py > $OUT/crc_bench.json 2>/dev/null
ls -la $OUT
