set -u
o=gpurun_out/rp14
mkdir -p $o
timeout 900 python -m pytest tests/test_gpu_rp_merge.py tests/test_gpu_rp_host.py tests/test_gpu_detres.py -q -x > $o/rp_tests.log 2>&1; echo "rc=$?" >> $o/rp_tests.log
tail -2 $o/rp_tests.log
for i in 1 2; do PIP_TIMING=1 timeout 600 python bench.py --op rp --steps 5 --warmup 3 --no-cpu --no-e2e >> $o/rp.json 2>> $o/rp.err; done
PIP_TIMING=1 timeout 600 python bench.py --op rp0 --steps 20 --warmup 5 --no-cpu --no-e2e >> $o/rp0.json 2>> $o/rp0.err
python tools/var_summary.py $o
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x -k "rp or perm" > $o/full_tests.log 2>&1; echo "rc=$?" >> $o/full_tests.log
tail -2 $o/full_tests.log
