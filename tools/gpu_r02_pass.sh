#!/bin/bash
# Round-2 GPU pass (re-entry): full GPU suite on the current code, smoke, small-N
# one-shot tiles, phase breakdown (variant build), sanitizers.
mkdir -p gpurun_out
python tools/build.py all > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
bash tools/build_variant.sh phases -DMOA_K1_PHASES > gpurun_out/build_phases.log 2>&1; echo "variant rc=$?"
timeout 1500 python -m pytest tests -q -m gpu -rf > gpurun_out/r02_gpu_all.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/r02_gpu_all.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_smoke.log 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/r02_smoke.log
timeout 600 python tools/small_n.py 128,256,384,512,768,1024 > gpurun_out/r02_small_n.json 2> gpurun_out/r02_small_n.err; echo "small_n rc=$?"; tail -c 1500 gpurun_out/r02_small_n.json
timeout 300 python tools/experiments/phases.py ab/libmoa_phases.so 128,256,512,1024 > gpurun_out/r02_phases.jsonl 2>&1; echo "phases rc=$?"; cat gpurun_out/r02_phases.jsonl
bash tools/gpu_sanitize.sh
