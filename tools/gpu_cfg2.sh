set -u
o=gpurun_out/cfg2
mkdir -p $o
for c in 17 25 26 27; do
  PIP_FILTER_CFG=$c timeout 600 python bench.py --op filter --steps 5 --warmup 3 --no-cpu --no-e2e > $o/filter_c$c.json 2> $o/filter_c$c.err
done
for c in 17 18 19; do
  PIP_SCAN_CFG=$c timeout 600 python bench.py --op scan --steps 5 --warmup 3 --no-cpu --no-e2e > $o/scan_c$c.json 2> $o/scan_c$c.err
done
PIP_FILTER_CFG=25 timeout 900 python -m pytest tests/test_gpu_scan_filter.py -q -x -k "filter" > $o/filter25_tests.log 2>&1; echo "rc=$?" >> $o/filter25_tests.log
PIP_SCAN_CFG=18 timeout 900 python -m pytest tests/test_gpu_scan_filter.py -q -x -k "scan" > $o/scan18_tests.log 2>&1; echo "rc=$?" >> $o/scan18_tests.log
PIP_TIMING=1 timeout 600 python bench.py --op rp --steps 3 --warmup 2 --no-cpu --no-e2e > $o/rp.json 2> $o/rp.err
PIP_TIMING=1 timeout 600 python bench.py --op rp0 --steps 5 --warmup 3 --no-cpu --no-e2e > $o/rp0.json 2> $o/rp0.err
timeout 900 python -m pytest tests/test_gpu_rp_merge.py tests/test_gpu_rp_host.py -q -x -k "rp" > $o/rp_tests.log 2>&1; echo "rc=$?" >> $o/rp_tests.log
