#!/usr/bin/env bash
# RP change check: permutation tests, then C0 bench lines with phase timers.
set -u
out=gpurun_out/${1:-rp_s3}
mkdir -p $out
timeout 900 python -m pytest tests -m gpu -x -q -k "rp or perm or c0 or c4 or detres" > $out/tests.log 2>&1; echo rc=$? >> $out/tests.log
for i in 1 2 3; do
  PIP_TIMING=1 timeout 300 python bench.py --op rp0 --steps 10 --warmup 3 --no-cpu --no-e2e > $out/rp0_$i.json 2> $out/rp0_$i.err
done
timeout 300 python bench.py --op rp0 --steps 10 --warmup 3 > $out/rp0_full.json 2> $out/rp0_full.err
tail -3 $out/tests.log
