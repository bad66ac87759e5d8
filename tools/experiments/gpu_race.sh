#!/bin/bash
mkdir -p gpurun_out
timeout 600 python tools/experiments/dbg_race2.py 200 > gpurun_out/race.log 2>&1
timeout 900 compute-sanitizer --tool racecheck --print-limit 10 python tools/experiments/dbg_race2.py 1 > gpurun_out/racecheck.log 2>&1
cat gpurun_out/race.log; grep -E "RACECHECK|hazard|Error|ERROR" gpurun_out/racecheck.log | head -10
