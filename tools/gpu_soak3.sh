set -u
o=gpurun_out/soak3
mkdir -p $o
timeout 900 python -m pytest tests/test_gpu_scan_filter.py tests/test_gpu_scan_filter_host.py tests/test_gpu_boundary.py tests/test_gpu_fullsize.py tests/test_distributed.py tests/test_sharded_abi.py -q -x -m gpu -k "scan or shard" > $o/scan_tests.log 2>&1; echo "rc=$?" >> $o/scan_tests.log; tail -2 $o/scan_tests.log
timeout 400 python tools/scan_soak.py 32 300 > $o/default_soak.log 2>&1; echo "rc=$?" >> $o/default_soak.log; tail -2 $o/default_soak.log
for i in 1 2; do timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e >> $o/s20.json 2>> $o/s20.err; done
timeout 600 python bench.py --op scan --steps 5 --warmup 3 --no-cpu --no-e2e >> $o/s5.json 2>> $o/s5.err
python tools/var_summary.py $o
