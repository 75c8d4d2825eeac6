python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "fused_subcycle" > gpurun_out/t4.log 2>&1
tail -2 gpurun_out/t4.log
timeout 300 python scripts/quick_perf.py hex2048 10 2>&1 | grep -v counts
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_fine_sub -s 2 -c 1 -o gpurun_out/sub_v2 -f python scripts/quick_perf.py hex2048 2 > gpurun_out/ncu_sub.log 2>&1
tail -3 gpurun_out/ncu_sub.log
