set -u
out=gpurun_out/ncu_sf
mkdir -p $out
full() {  # op log2n kernel-regex
  local cmd="python tools/profile_op.py --op $1 --log2n $2 --reps 2"
  $cmd > $out/profile_op_$1.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:$3 -s 1 -c 1 \
      -o $out/full_$1 $cmd > $out/ncu_full_$1.log 2>&1
}
full scan 28 scan_ws2
full filter 28 filter_ws2
for op in scan filter; do
  cmd="python bench.py --op $op --steps 2 --warmup 3 --no-cpu --no-e2e"
  $cmd > $out/plain_$op.json 2> $out/plain_$op.err && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file $out/launches_$op.csv $cmd > /dev/null 2> $out/ncu_launch_$op.err
done
ls -la $out
for op in scan filter; do
  python tools/ncu_summary.py $out/full_$op.ncu-rep 10 > $out/ncu_${op}_summary.txt 2>&1
  python tools/launch_summary.py $out/launches_$op.csv 5 > $out/launches_${op}_summary.txt 2>&1
done
rm -f $out/*.ncu-rep
ls -la $out
