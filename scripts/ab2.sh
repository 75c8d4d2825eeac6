#!/bin/bash
# scripts/ab2.sh: like ab.sh, but every variant is "NVCC_EXTRA|ENV=VAL ..." (env applied to the run)
CFG=config5
if [ "$1" == "--config" ]; then CFG=$2; shift 2; fi
for V in "$@"; do
  EXTRA="${V%%|*}"; ENVS="${V#*|}"; [ "$ENVS" == "$V" ] && ENVS=""
  FBLTS_NVCC_EXTRA="$EXTRA" python -m paper_2405_10505_b200.build --force > /dev/null 2>&1 || { echo "build failed: $V"; continue; }
  env $ENVS timeout 300 python bench.py --config $CFG --no-cpu-baseline --no-e2e --no-global --steps 10 > gpurun_out/ab.log 2>&1
  echo "=== variant [$EXTRA] env [$ENVS]"
  python - <<'PY'
import json
lines = open("gpurun_out/ab.log").read().strip().splitlines()
try:
    d = json.loads(lines[-1])
except Exception:
    print("\n".join(lines[-15:])); raise SystemExit
print(f"ms/step {d['ms_per_step']:.3f}  value {d['value']:.4e}  step_frac {d['roofline']['step_frac']:.3f}")
for k, v in d["kernels"].items():
    print(f"  {k:11s} {v['ms_per_launch']:.4f} ms x{v['launches_per_step']:.0f}  {v['GBps']:.0f} GB/s")
PY
done
