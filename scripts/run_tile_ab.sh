#!/bin/bash
# A/B of the staged tile size / ring depth / launch split on hex2048 (quick_perf), then restore the default build.
for V in "$@"; do
  FBLTS_NVCC_EXTRA="$V" python -m paper_2405_10505_b200.build --force > /dev/null 2>&1 || { echo "build failed: $V"; continue; }
  for SPLIT in 0 1; do
    echo "=== [$V] SPLIT=$SPLIT"
    FBLTS_SPLIT=$SPLIT timeout 300 python scripts/quick_perf.py hex2048 10 2>&1 | grep -E "ms/coarse|fine_s2|fine_s3|vel_s1|tile_smem" | sed 's/counts=.*tile_smem_bytes/tile_smem_bytes/; s/, .sub_tiles.*//'
  done
done
python -m paper_2405_10505_b200.build --force > /dev/null 2>&1
