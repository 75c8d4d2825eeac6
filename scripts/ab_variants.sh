#!/bin/bash
# Development A/B over build variants: AB_VARIANTS="label|nvcc extra|env;label|...", AB_CFG (config).
# Prints ms per step and per-kind times; ends with the default build restored.
CFG=${AB_CFG:-config5_2048}
IFS=';' read -ra VS <<< "$AB_VARIANTS"
for v in "${VS[@]}"; do
  IFS='|' read -r lab extra envs <<< "$v"
  FBLTS_NVCC_EXTRA="$extra" python -m paper_2405_10505_b200.build --force > gpurun_out/build_$lab.log 2>&1 || { echo "build $lab failed"; continue; }
  for cfg in $CFG; do
    env $envs timeout 900 python bench.py --config $cfg --steps ${AB_STEPS:-20} --no-cpu-baseline --no-e2e --no-global \
       > gpurun_out/ab_${lab}_$cfg.log 2>&1
    grep '^{' gpurun_out/ab_${lab}_$cfg.log | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); k=d['kernels']
print('$lab $cfg ms/step %.3f'%d['ms_per_step'], ' '.join('%s=%.3f'%(n,v['ms_per_step']) for n,v in sorted(k.items()) if v['ms_per_step']>0.05), 'dom', d['roofline']['kernel'], '%.3f'%d['roofline']['frac'], 'step %.3f'%d['roofline']['step_frac'])" || tail -3 gpurun_out/ab_${lab}_$cfg.log
  done
done
python -m paper_2405_10505_b200.build --force > /dev/null 2>&1
