#!/bin/bash
# Session re-entry check: rebuild, smoke, full GPU suite, the default bench line.
mkdir -p gpurun_out
python tools/build.py all > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/v_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/v_smoke.log
timeout 2400 python -m pytest tests -q -m gpu -rf > gpurun_out/v_gpu_all.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/v_gpu_all.log
timeout 1500 python bench.py > gpurun_out/v_bench.json 2> gpurun_out/v_bench.err; echo "bench rc=$?"; head -c 800 gpurun_out/v_bench.json; echo
