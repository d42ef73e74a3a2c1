#!/usr/bin/env bash
# One-call profile sweep for the round's evidence (run under gpurun):
#   launch lists of each bench command (ncu --metrics gpu__time_duration.sum)
#   and one `ncu --set full` capture of each op's dominant kernel.
# Every ncu command is preceded by the same command run without ncu (&&).
set -u
out=gpurun_out
mkdir -p $out
for op in scan filter merge rp rp0; do
  cmd="python bench.py --op $op --steps 2 --warmup 3 --no-cpu --no-e2e"
  $cmd > $out/plain_$op.json 2> $out/plain_$op.err && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file $out/launches_$op.csv $cmd > /dev/null 2> $out/ncu_launch_$op.err
done
full() {  # op log2n kernel-regex
  local cmd="python tools/profile_op.py --op $1 --log2n $2 --reps 2"
  $cmd > /dev/null 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:$3 -s 1 -c 1 \
      -o $out/full_$1 $cmd > $out/ncu_full_$1.log 2>&1
}
full scan 28 scan_ws2
full filter 28 filter_ws2
full merge 28 merge_kernel
full rp 26 rp_kernel
ls -la $out
