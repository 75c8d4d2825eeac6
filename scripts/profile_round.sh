#!/bin/bash
# Evidence for profiles/ (round ${ROUND:-r2}): the bench line, the launch list of the bench command
# (per-launch device times, cold-cache and serialised under ncu: compare shares), and one
# --set full capture of a config-5 coarse step (every kernel kind), summarised as CSV.
R=${ROUND:-r2}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python bench.py > gpurun_out/${R}_bench.log 2>&1
grep '^{' gpurun_out/${R}_bench.log | tail -1 > gpurun_out/${R}_bench.json
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-global > gpurun_out/${R}_plain.log 2>&1 &&
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
  --log-file gpurun_out/${R}_launches_config5.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-global \
  > gpurun_out/${R}_ncu_launch.log 2>&1
timeout 300 python scripts/one_step.py config5 3 > gpurun_out/${R}_one_step.log 2>&1 &&
timeout 1800 ncu --set full --clock-control none --import-source on -s 50 -c 45 -o gpurun_out/${R}_step_full -f \
  python scripts/one_step.py config5 3 > gpurun_out/${R}_ncu_full.log 2>&1
tail -2 gpurun_out/${R}_ncu_full.log
ncu -i gpurun_out/${R}_step_full.ncu-rep --page raw --csv > gpurun_out/${R}_step_full_raw.csv 2>/dev/null
ncu -i gpurun_out/${R}_step_full.ncu-rep --page details --csv > gpurun_out/${R}_step_full_details.csv 2>/dev/null
rm -f gpurun_out/${R}_step_full.ncu-rep
ls -la gpurun_out | tail -12
