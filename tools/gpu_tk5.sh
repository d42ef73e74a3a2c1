set -u
o=gpurun_out/tk5
mkdir -p $o
for rep in 1 2 3; do
  for cfg in 21 25 28 29; do
    PIP_SCAN_CFG=$cfg timeout 600 python bench.py --op scan --steps 10 --warmup 3 --no-cpu --no-e2e >> $o/cfg$cfg.json 2>> $o/cfg$cfg.err
  done
done
for cfg in 21 25; do
  PIP_SCAN_CFG=$cfg timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e >> $o/s20_cfg$cfg.json 2>> $o/s20_cfg$cfg.err
done
python tools/var_summary.py $o
PIP_SCAN_CFG=25 timeout 900 python -m pytest tests/test_gpu_scan_filter.py tests/test_gpu_scan_filter_host.py tests/test_gpu_boundary.py -q -x -k "scan" > $o/scan_tests.log 2>&1; echo "rc=$?" >> $o/scan_tests.log
tail -2 $o/scan_tests.log
