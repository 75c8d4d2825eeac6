#!/bin/bash
# development A/B of compile-time knobs on a 2048^2 block of the config-5 recipe
for x in ${VARIANTS:-"-DFBLTS_MINB=1" "-DFBLTS_MINB=6" "-DFBLTS_MINB=8"}; do
  echo "== $x"
  FBLTS_NVCC_EXTRA="$x" python -m paper_2405_10505_b200.build --force > /dev/null
  python scripts/quick_perf.py hex2048 10 2>&1 | grep -E "ms/coarse|fine_|coarse_s"
done
python -m paper_2405_10505_b200.build --force > /dev/null
