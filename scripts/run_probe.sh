python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests -m gpu -q -x -k "not config5_full" > gpurun_out/t10.log 2>&1; tail -2 gpurun_out/t10.log
for V in 0 1; do echo "== FBLTS_SLOWPRE_CELL=$V"; FBLTS_SLOWPRE_CELL=$V timeout 300 python scripts/quick_perf.py hex2048 10 2>&1 | grep -E "ms/coarse|slow_pre|slow_edge"; done
timeout 900 python bench.py > gpurun_out/bench.log 2>&1
grep '^{' gpurun_out/bench.log | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('ms/step', d['ms_per_step'], 'value', d['value'], 'e2e', d['e2e']['value'], d['roofline']['kernel'], d['roofline']['frac'], d['roofline']['step_frac']); print({k:(round(v['ms_per_step'],3), round(v['GBps'])) for k,v in d['kernels'].items()})"
