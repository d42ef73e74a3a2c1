#!/usr/bin/env bash
# One-call profile sweep for the round's evidence (run under gpurun):
#   bench lines of every op, launch lists of each bench command (ncu
#   --metrics gpu__time_duration.sum) and ncu captures of the dominant
#   kernels.  Every ncu command is preceded by the same command run without
#   ncu (&&).
set -u
out=gpurun_out/${1:-prof}
mkdir -p $out
nvidia-smi > $out/gpu.txt 2>&1
for op in scan filter merge rp rp0 partition; do
  timeout 900 python bench.py --op $op --steps 5 --warmup 3 > $out/bench_$op.json 2> $out/bench_$op.err
done
timeout 600 python bench.py > $out/bench_default.json 2> $out/bench_default.err
for op in scan filter merge rp rp0; do
  timeout 600 python bench.py --op $op --impl reference --steps 3 --warmup 1 > $out/ref_$op.json 2> $out/ref_$op.err
done
for op in scan filter merge rp rp0; do
  cmd="python bench.py --op $op --steps 2 --warmup 3 --no-cpu --no-e2e"
  $cmd > $out/plain_$op.json 2> $out/plain_$op.err && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file $out/launches_$op.csv $cmd > /dev/null 2> $out/ncu_launch_$op.err
done
full() {  # op log2n kernel-regex [extra ncu args]
  local cmd="python tools/profile_op.py --op $1 --log2n $2 --reps 2"
  $cmd > $out/profile_op_$1.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:$3 -s 1 -c 1 \
      -o $out/full_$1 $cmd > $out/ncu_full_$1.log 2>&1
}
full scan 28 scan_ws2
full filter 28 filter_ws2
full merge 28 merge_kernel
full rmw 30 random_rmw
full rmwx 30 random_rmw
cmd="python tools/profile_op.py --op rp --log2n 30 --reps 1"
$cmd > $out/profile_op_rp.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct \
    --clock-control none -k regex:rp_kernel --csv --log-file $out/rp30_ncu.csv $cmd > $out/ncu_rp30.log 2>&1
ls -la $out
