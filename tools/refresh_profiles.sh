#!/bin/bash
# One GPU call that regenerates the committed measurement artefacts (run under gpurun):
#   bench line, cfg1/3/5 DAS throughput, the bench launch list, ncu --set full of
#   K1 / K2 / the row operator. Outputs land in gpurun_out/; copy to profiles/<round>/.
set -x
python bench.py > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err
python tools/bench_configs.py > gpurun_out/bench_configs.jsonl 2> gpurun_out/bench_configs.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline \
  > gpurun_out/ncu_launches.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"das_image|analytic|rowconv_tc1" -c 3 \
  -o gpurun_out/prof_full python tools/profile_kernels.py --frames 64 --maps 256 > gpurun_out/ncu_full.log 2>&1
ls -la gpurun_out
