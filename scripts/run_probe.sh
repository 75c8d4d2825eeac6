python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "unfused" > gpurun_out/t16.log 2>&1; tail -2 gpurun_out/t16.log
for V in "" "-DFBLTS_WS_CG=4" "-DFBLTS_WS_CW=24 -DFBLTS_WS_CG=3 -DFBLTS_WS_NB=3"; do
  FBLTS_NVCC_EXTRA="$V" python -m paper_2405_10505_b200.build --force > /dev/null 2>&1 || { echo "build failed: $V"; continue; }
  for W in 0 1; do
    [ "$W" == "0" ] && [ -n "$V" ] && continue
    echo "=== [$V] WS=$W"
    FBLTS_WS=$W timeout 300 python scripts/quick_perf.py hex2048 10 2>&1 | grep -E "ms/coarse|fine_s2|fine_s3|vel_s1|coarse_s|Error"
  done
done
python -m paper_2405_10505_b200.build --force > /dev/null 2>&1
