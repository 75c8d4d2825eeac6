#!/bin/bash
# Evidence for profiles/: launch list of the bench command (per-launch device times, cold-cache and
# serialised under ncu) and one --set full capture of a config-5 coarse step (every kernel kind).
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python bench.py > gpurun_out/bench_final.log 2>&1
grep '^{' gpurun_out/bench_final.log | tail -1 > gpurun_out/bench_final.json
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv \
  --log-file gpurun_out/launches_v4.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-global \
  > gpurun_out/ncu_launch.log 2>&1
# one coarse step under --set full: skip the set_state / warm-up launches, capture 40 launches
timeout 1500 ncu --set full --clock-control none --import-source on -s 60 -c 40 -o gpurun_out/step_full -f \
  python scripts/one_step.py config5 3 > gpurun_out/ncu_full.log 2>&1
tail -2 gpurun_out/ncu_full.log
# keep the merge-back small: tables only
ncu -i gpurun_out/step_full.ncu-rep --page raw --csv > gpurun_out/step_full_raw.csv 2>/dev/null
ncu -i gpurun_out/step_full.ncu-rep --page details --csv > gpurun_out/step_full_details.csv 2>/dev/null
rm -f gpurun_out/step_full.ncu-rep
ls -la gpurun_out
