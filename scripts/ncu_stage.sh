#!/bin/bash
# ncu --set full of the deep stage-3 sweep, both tile kernels, on a 2048^2 config-5 block.
python -m paper_2405_10505_b200.build > gpurun_out/build.log 2>&1 || exit 1
for d in 0 1; do
  FBLTS_DIRECT=$d timeout 300 python scripts/one_step.py config5_2048 2 > gpurun_out/plain_$d.log 2>&1 &&
  FBLTS_DIRECT=$d timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_stage_ -s 6 -c 2 \
      -o gpurun_out/stage_$d -f python scripts/one_step.py config5_2048 2 > gpurun_out/ncu_$d.log 2>&1
  tail -3 gpurun_out/ncu_$d.log
done
