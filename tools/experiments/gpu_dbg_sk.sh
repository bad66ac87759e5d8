#!/bin/bash
for c in "8192 128 128 6 2" "2048 64 64 4 2" "1024 64 64 4 2" "3072 128 128 6 2" "1280 128 64 4 2 x 148"; do
  echo "== $c"; timeout 300 python tools/experiments/dbg_sk.py $c 2>&1 | grep -E "^rep|kind" | cut -c1-300
done
