python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests -m gpu -q -x -k "unfused or config2 or parity_100 or other_M" > gpurun_out/t29.log 2>&1; tail -2 gpurun_out/t29.log
for V in 0 1; do echo "== FBLTS_BAND_SIDE=$V"; FBLTS_BAND_SIDE=$V timeout 300 python scripts/quick_perf.py hex2048 20 2>&1 | grep -E "ms/coarse"; done
for V in 0 1; do echo "== FBLTS_BAND_SIDE=$V"; FBLTS_BAND_SIDE=$V timeout 600 python bench.py --no-cpu-baseline --no-global --no-e2e --steps 50 2>&1 | grep '^{' | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('config5 ms/step', d['ms_per_step'], d['value'])"; done
