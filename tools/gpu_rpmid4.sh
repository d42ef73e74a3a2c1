set -u
o=gpurun_out/rpmid4
mkdir -p $o
for lg in 24 25 26 27; do
  for l1 in 0 1; do
    PIP_RP_LARGE1=$l1 PIP_TIMING=1 timeout 600 python bench.py --op rp --log2n $lg --steps 5 --warmup 2 --no-cpu --no-e2e >> $o/lg${lg}_large$l1.json 2>> $o/lg${lg}_large$l1.err
  done
done
python tools/var_summary.py $o
timeout 900 python -m pytest tests/test_gpu_rp_merge.py -q -x -k "reservation_modes" > $o/rp_tests.log 2>&1; echo "rc=$?" >> $o/rp_tests.log
tail -2 $o/rp_tests.log
