set -u
o=gpurun_out/rp10
mkdir -p $o
timeout 900 python -m pytest tests/test_gpu_rp_merge.py tests/test_gpu_rp_host.py tests/test_gpu_detres.py -q -x > $o/rp_tests.log 2>&1; echo "rc=$?" >> $o/rp_tests.log
tail -3 $o/rp_tests.log
for d in 0 4 0 4; do
  PIP_RP_DBG=$d PIP_TIMING=1 timeout 600 python bench.py --op rp --steps 3 --warmup 2 --no-cpu --no-e2e >> $o/dbg$d.json 2>> $o/dbg$d.err
done
python tools/var_summary.py $o
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x -k "rp or perm" > $o/full_tests.log 2>&1; echo "rc=$?" >> $o/full_tests.log
tail -3 $o/full_tests.log
