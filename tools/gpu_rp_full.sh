set -u
o=gpurun_out/rpfull
mkdir -p $o
cmd="python tools/profile_op.py --op rp --log2n 30 --reps 1"
$cmd > $o/profile_op_rp.log 2>&1 && \
timeout 3000 ncu --set full --clock-control none --import-source on -k regex:rp_kernel -c 1 -o $o/full_rp $cmd > $o/ncu_full_rp.log 2>&1
tail -3 $o/ncu_full_rp.log
ls -la $o
