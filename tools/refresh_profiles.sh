#!/bin/bash
# One GPU call that regenerates the committed measurement artefacts (run under gpurun):
#   bench line, the bench launch list, ncu --set full of K1 / K2 / the row
#   operator / K5. Outputs land in gpurun_out/; copy to profiles/<round>/.
set -x
python bench.py > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline \
  > gpurun_out/ncu_launches.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"das_image|analytic|rowconv_tc1|row_psf" -c 4 \
  -o gpurun_out/prof_full python tools/profile_kernels.py --frames 256 --maps 256 > gpurun_out/ncu_full.log 2>&1
ls -la gpurun_out
