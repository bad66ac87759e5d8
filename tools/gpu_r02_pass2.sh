#!/bin/bash
# Round-2 pass 2: full GPU suite on the static-schedule/gate/lag K1 (K5 removed), the
# latency-tile chooser, the 64x64 regression check against the round-1 build,
# sanitizers, and the raster group under the wave gate at 32768^3.
mkdir -p gpurun_out/sanitizer
python tools/build.py all > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_smoke.log 2>&1; rc=$?; echo "smoke rc=$rc"; tail -2 gpurun_out/r02_smoke.log; [ $rc -ne 0 ] && exit 1
timeout 1800 python -m pytest tests -q -m gpu -rf > gpurun_out/r02_gpu_all.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/r02_gpu_all.log
timeout 600 python tools/small_n.py 64,128,192,256,320,384,448,512,768,1024 > gpurun_out/r02_small_n.json 2> gpurun_out/r02_small_n.err; echo "small_n rc=$?"; cat gpurun_out/r02_small_n.err | python -c "
import sys, json
for l in sys.stdin:
    try: d = json.loads(l)
    except Exception: continue
    best = sorted((c.get('graph_us', 1e9), c['cfg'][1:]) for c in d['cfgs'])
    ch = [c.get('graph_us') for c in d['cfgs'] if c['cfg'][1:] == d['chosen'][1:]]
    print(d['N'], 'chosen', d['chosen'][1:], ch, 'best', best[:3])
"
AB_ROUNDS=3 timeout 900 python tools/experiments/ab_shapes.py "768,768,768;1024,1024,1024;1536,1536,1536;2048,2048,2048;4096,4096,4096" ab/libmoa_r01.so paper_2306_11148_b200/libmoa.so > gpurun_out/r02_ab_r01.jsonl 2>&1; echo "ab r01 rc=$?"; cut -c1-300 gpurun_out/r02_ab_r01.jsonl
for t in racecheck memcheck synccheck; do
  timeout 1500 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize_run.py > gpurun_out/sanitizer/r02_$t.log 2>&1
  echo "$t rc=$?"; tail -3 gpurun_out/sanitizer/r02_$t.log
done
ROUNDS=2 timeout 900 python tools/experiments/energy_traffic.py 32768 8,12,16 > gpurun_out/r02_raster_32768.jsonl 2>&1; echo "raster rc=$?"; cat gpurun_out/r02_raster_32768.jsonl
RASTER_NCU=1 timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:k_dgemm_tma -s 1 --csv --log-file gpurun_out/r02_raster_ncu_32768.csv python tools/experiments/energy_traffic.py 32768 8,12,16 > /dev/null 2>&1; echo "ncu raster rc=$?"
