for V in "-DFBLTS_PROBE=1" "-DFBLTS_PROBE=3" "-DFBLTS_PROBE=4"; do
  FBLTS_NVCC_EXTRA="$V" python -m paper_2405_10505_b200.build --force > /dev/null 2>&1 || { echo "build failed: $V"; continue; }
  echo "=== [$V]"
  timeout 300 python scripts/quick_perf.py hex2048 10 2>&1 | grep -E "ms/coarse|fine_s2|fine_s3|vel_s1|FbltsError"
done
python -m paper_2405_10505_b200.build --force > /dev/null 2>&1
