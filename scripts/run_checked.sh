#!/bin/bash
# GPU suite on a bounds-checked build (FBLTS_CHECK=1: every shared-memory index derived from the tile
# tables is verified on the device; a violation traps), then the default build is restored.
FBLTS_NVCC_EXTRA="-DFBLTS_CHECK=1" python -m paper_2405_10505_b200.build --force > gpurun_out/build_check.log 2>&1 || exit 1
timeout 2400 python -m pytest tests -m gpu -q -x -k "not bench_contract" > gpurun_out/gpu_tests_checked.log 2>&1   # bench.py refuses CHECK builds
tail -3 gpurun_out/gpu_tests_checked.log
python -m paper_2405_10505_b200.build --force > /dev/null 2>&1
