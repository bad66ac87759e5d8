#!/bin/bash
# Late round-2 final pass: full GPU suite, smoke, the driver bench line + its ncu launch
# list, ncu of configs[0] (one-shot latency tile) and configs[3], per-config numbers,
# chooser sweep, sanitizers.
mkdir -p gpurun_out/sanitizer
python tools/build.py all > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f2_smoke.log 2>&1; rc=$?; echo "smoke rc=$rc"; tail -2 gpurun_out/f2_smoke.log; [ $rc -ne 0 ] && exit 1
timeout 2400 python -m pytest tests -q -m gpu -rf > gpurun_out/f2_gpu_all.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/f2_gpu_all.log
timeout 1500 python bench.py > gpurun_out/f2_bench.json 2> gpurun_out/f2_bench.err; echo "bench rc=$?"; head -c 400 gpurun_out/f2_bench.json; echo
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/f2_launches_bench.csv python bench.py --steps 2 --warmup 1 --no-sweep --no-cpu --no-e2e --no-variants > gpurun_out/f2_launches_bench.log 2>&1; echo "launches rc=$?"
python tools/ncu_summary.py launches gpurun_out/f2_launches_bench.csv > gpurun_out/f2_launches_bench.json 2>/dev/null
bash tools/gpu_prof_configs.sh c0 c3
timeout 900 python tools/bench_configs.py --sections c0,c3 --skip-blocks > gpurun_out/f2_configs.json 2> gpurun_out/f2_configs.err; echo "configs rc=$?"
timeout 900 python tools/experiments/chooser_sweep.py > gpurun_out/f2_chooser_sweep.jsonl 2> gpurun_out/f2_chooser_sweep.err; echo "chooser rc=$?"; tail -2 gpurun_out/f2_chooser_sweep.jsonl
for t in racecheck memcheck synccheck; do
  timeout 1500 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize_run.py > gpurun_out/sanitizer/f2_$t.log 2>&1
  echo "$t rc=$?"; tail -1 gpurun_out/sanitizer/f2_$t.log
done
