#!/bin/bash
# Quick measurement of the current build: bench on a config-5 block and on config 5, kernel table.
python -m paper_2405_10505_b200.build > gpurun_out/build.log 2>&1 || exit 1
for cfg in ${QCFGS:-config5_2048 config5}; do
  env $QENV timeout 900 python bench.py --config $cfg --steps 20 --no-cpu-baseline --no-e2e --no-global > gpurun_out/q_$cfg.log 2>&1
  grep '^{' gpurun_out/q_$cfg.log | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); k=d['kernels']
print('$cfg ms/step %.3f'%d['ms_per_step'], ' '.join('%s=%.3f'%(n,v['ms_per_step']) for n,v in sorted(k.items()) if v['ms_per_step']>0.05), 'dom', d['roofline']['kernel'], '%.3f'%d['roofline']['frac'], 'step %.3f'%d['roofline']['step_frac'])"
done
