#!/bin/bash
# Development A/B of the fused-subcycle kernel: rebuild with each FBLTS_NVCC_EXTRA variant and time
# scripts/quick_perf.py on a hex mesh (default hex2048), with and without the fused subcycle.
MESH=${MESH:-hex2048}
for V in "$@"; do
  FBLTS_NVCC_EXTRA="$V" python -m paper_2405_10505_b200.build --force > /dev/null 2>&1 || { echo "build failed: $V"; continue; }
  echo "=== variant [$V]"
  timeout 300 python scripts/quick_perf.py $MESH 10 2>&1 | grep -v counts
done
