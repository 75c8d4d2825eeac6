python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests/test_bench_contract.py -q -m gpu > gpurun_out/t39.log 2>&1; tail -3 gpurun_out/t39.log
