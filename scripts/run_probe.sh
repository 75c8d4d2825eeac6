python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests -m gpu -q -x -k "unsplit or energy or refresh" > gpurun_out/t12.log 2>&1; tail -2 gpurun_out/t12.log
