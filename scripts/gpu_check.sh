#!/bin/bash
# Parity on the GPU (the fast parity tests + the full-length goldens of configs 1, 2 and 5) and a config-5
# bench A/B: RUNS="ENV=.. ENV2=.." (one bench per entry, "-" for the default build).
mkdir -p gpurun_out
summ() {
  grep '^{' $1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); k=d['kernels']
print('$2 ms/step %.3f'%d['ms_per_step'], ' '.join('%s=%.3f'%(n,v['ms_per_step']) for n,v in sorted(k.items()) if v['ms_per_step']>0.05), 'dom', d['roofline']['kernel'], '%.3f'%d['roofline']['frac'], 'step %.3f'%d['roofline']['step_frac'])"
}
if [ -z "$NOTEST" ]; then
  timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_full.py -x -q -m gpu -k "${TESTK:-not config5_full_size and not config4}" > gpurun_out/gpu_check_tests.log 2>&1
  echo "tests: $(tail -1 gpurun_out/gpu_check_tests.log)"
  grep -E "FAILED|Error" gpurun_out/gpu_check_tests.log | head -5
fi
for v in ${RUNS:--}; do
  env ${v#-} timeout 900 python bench.py --steps 20 --no-cpu-baseline --no-e2e --no-global > gpurun_out/gpu_check_bench.log 2>&1
  summ gpurun_out/gpu_check_bench.log "$v"
done
