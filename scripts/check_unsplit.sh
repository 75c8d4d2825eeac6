#!/bin/bash
# Parity of the unsplit / slow-sweep changes and the config-5 benches (split A/B of FBLTS_VF, unsplit).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/cu_build.log 2>&1 || { tail gpurun_out/cu_build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "unsplit or vorticity or energy or hurricane or rk4 or rk32 or 100_steps or sphere or config3 or config2" > gpurun_out/cu_tests.log 2>&1
echo "tests: $(tail -1 gpurun_out/cu_tests.log)"; grep -E "^FAILED|Error" gpurun_out/cu_tests.log | head -5
NOTEST=1 RUNS="- FBLTS_VF=0" bash scripts/gpu_check.sh
timeout 900 python bench.py --unsplit --steps 10 --no-cpu-baseline --no-e2e --no-global > gpurun_out/cu_unsplit.log 2>&1
grep '^{' gpurun_out/cu_unsplit.log | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); k=d['kernels']
print('unsplit ms/step %.3f'%d['ms_per_step'], ' '.join('%s=%.3f'%(n,v['ms_per_step']) for n,v in sorted(k.items()) if v['ms_per_step']>0.05), 'dom', d['roofline']['kernel'], '%.3f'%d['roofline']['frac'], 'step %.3f'%d['roofline']['step_frac'])"
