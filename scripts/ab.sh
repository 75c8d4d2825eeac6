#!/bin/bash
# Development A/B timing on the GPU box: rebuild libfblts.so with each FBLTS_NVCC_EXTRA variant
# given as an argument ("" = default) and print the bench's per-kernel summary for each.
# Usage: scripts/ab.sh [--config config5] "" "-DFOO=1" ...
CFG=config5
if [ "$1" == "--config" ]; then CFG=$2; shift 2; fi
for V in "$@"; do
  FBLTS_NVCC_EXTRA="$V" python -m paper_2405_10505_b200.build --force > /dev/null 2>&1 || { echo "build failed: $V"; continue; }
  timeout 300 python bench.py --config $CFG --no-cpu-baseline --no-e2e --no-global --steps 10 > gpurun_out/ab.log 2>&1
  echo "=== variant [$V] ${FBLTS_TILED:+TILED=$FBLTS_TILED}"
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
