python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 600 python -m pytest tests -m gpu -q -x -k "diagnostics or conservation or set_state or dist" > gpurun_out/t6.log 2>&1; tail -2 gpurun_out/t6.log
timeout 300 python scripts/e2e_parts.py 4096
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_stage_tiled -s 6 -c 1 -o gpurun_out/tiled_s3 -f python scripts/quick_perf.py hex2048 1 > gpurun_out/ncu_tiled.log 2>&1
tail -2 gpurun_out/ncu_tiled.log
