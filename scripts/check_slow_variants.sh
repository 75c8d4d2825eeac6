#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "unsplit or vorticity or energy or refresh or hurricane" > gpurun_out/cu3_tests.log 2>&1
echo "tests: $(tail -1 gpurun_out/cu3_tests.log)"; grep -E "^FAILED|Error" gpurun_out/cu3_tests.log | head -5
for a in "--unsplit" "--slow-refresh"; do
for v in - FBLTS_VF=0; do
env ${v#-} timeout 900 python bench.py $a --steps 10 --no-cpu-baseline --no-e2e --no-global > gpurun_out/cu3_b.log 2>&1
grep '^{' gpurun_out/cu3_b.log | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); k=d['kernels']
print('$a $v ms/step %.3f'%d['ms_per_step'], ' '.join('%s=%.3f'%(n,v['ms_per_step']) for n,v in sorted(k.items()) if v['ms_per_step']>0.05), 'dom', d['roofline']['kernel'], '%.3f'%d['roofline']['frac'], 'step %.3f'%d['roofline']['step_frac'])"
done; done
