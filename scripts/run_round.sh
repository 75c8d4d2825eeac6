#!/bin/bash
# Round check on the GPU box: build, GPU tests, smoke, default bench line (gpurun_out/).
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1 || { tail -20 gpurun_out/smoke.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q -x --durations=10 ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/gpu_tests.log 2>&1
tail -15 gpurun_out/gpu_tests.log
[ -n "$NO_BENCH" ] && exit 0
timeout 900 python bench.py > gpurun_out/bench.log 2>&1
grep '^{' gpurun_out/bench.log | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('ms/step', d['ms_per_step'], 'value', d['value'], 'e2e', d['e2e']['value'], d['roofline']['kernel'], d['roofline']['frac'], d['roofline']['step_frac'])"
