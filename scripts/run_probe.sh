python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests -m gpu -q -x -k "fused_subcycle" -rs > gpurun_out/t24.log 2>&1; tail -4 gpurun_out/t24.log
