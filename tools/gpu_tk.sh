set -u
o=gpurun_out/tk
mkdir -p $o
PIP_SCAN_CFG=21 timeout 900 python -m pytest tests/test_gpu_scan_filter.py -q -x -k "scan" > $o/scan_tests.log 2>&1; echo "rc=$?" >> $o/scan_tests.log
tail -2 $o/scan_tests.log
for rep in 1 2 3; do
  for cfg in 17 21; do
    PIP_SCAN_CFG=$cfg timeout 600 python bench.py --op scan --steps 10 --warmup 3 --no-cpu --no-e2e >> $o/cfg$cfg.json 2>> $o/cfg$cfg.err
  done
done
python tools/var_summary.py $o
