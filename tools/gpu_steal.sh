set -u
o=gpurun_out/steal
mkdir -p $o
for pct in 0 10 20 30 50 100; do
  PIP_RP_STEAL=$pct PIP_TIMING=1 timeout 600 python bench.py --op rp --steps 3 --warmup 2 --no-cpu --no-e2e >> $o/steal$pct.json 2>> $o/steal$pct.err
done
python tools/var_summary.py $o
PIP_RP_STEAL=25 timeout 900 python -m pytest tests/test_gpu_rp_merge.py -q -x -k "reservation_modes or golden or vs_oracle" > $o/rp_tests.log 2>&1; echo "rc=$?" >> $o/rp_tests.log
tail -2 $o/rp_tests.log
