#!/bin/bash
# Last confirmation of the committed tree: smoke, full GPU suite, the driver bench line.
mkdir -p gpurun_out
python tools/build.py all > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f4_smoke.log 2>&1; rc=$?; echo "smoke rc=$rc"; tail -1 gpurun_out/f4_smoke.log; [ $rc -ne 0 ] && exit 1
timeout 2400 python -m pytest tests -q -m gpu -rf > gpurun_out/f4_gpu_all.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/f4_gpu_all.log
timeout 1500 python bench.py > gpurun_out/f4_bench.json 2> gpurun_out/f4_bench.err; echo "bench rc=$?"; head -c 300 gpurun_out/f4_bench.json; echo
