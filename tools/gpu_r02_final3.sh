#!/bin/bash
# Confirmation after the opaque-address K1 change and the chooser factor: smoke, full GPU
# suite, the bench line, chooser sweep, small-N table.
mkdir -p gpurun_out
python tools/build.py all > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f3_smoke.log 2>&1; rc=$?; echo "smoke rc=$rc"; tail -1 gpurun_out/f3_smoke.log; [ $rc -ne 0 ] && exit 1
timeout 2400 python -m pytest tests -q -m gpu -rf > gpurun_out/f3_gpu_all.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/f3_gpu_all.log
timeout 1500 python bench.py > gpurun_out/f3_bench.json 2> gpurun_out/f3_bench.err; echo "bench rc=$?"; head -c 300 gpurun_out/f3_bench.json; echo
timeout 900 python tools/experiments/chooser_sweep.py > gpurun_out/f3_chooser_sweep.jsonl 2> gpurun_out/f3_chooser_sweep.err; echo "chooser rc=$?"
timeout 600 python tools/small_n.py 64,128,192,256,320,384,448,512,640,768,1024 > gpurun_out/f3_small_n.json 2> gpurun_out/f3_small_n.err; echo "small_n rc=$?"
