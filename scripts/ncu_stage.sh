#!/bin/bash
# ncu --set full (with source) of the deep stage-3 sweep on a 2048^2 config-5 block; CSV exports only.
python -m paper_2405_10505_b200.build > gpurun_out/build.log 2>&1 || exit 1
timeout 300 python scripts/one_step.py config5_2048 2 > gpurun_out/plain_s.log 2>&1 &&
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_stage_tiled -s 5 -c 1 \
    -o gpurun_out/stage_s -f python scripts/one_step.py config5_2048 2 > gpurun_out/ncu_s.log 2>&1
ncu -i gpurun_out/stage_s.ncu-rep --page source --csv --print-source sass > gpurun_out/stage_s_sass.csv 2>/dev/null
ncu -i gpurun_out/stage_s.ncu-rep --page raw --csv > gpurun_out/stage_s_raw.csv 2>/dev/null
rm -f gpurun_out/stage_s.ncu-rep
tail -2 gpurun_out/ncu_s.log
