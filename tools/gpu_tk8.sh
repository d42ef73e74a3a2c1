set -u
o=gpurun_out/tk8
mkdir -p $o
PIP_FILTER_CFG=41 timeout 900 python -m pytest tests/test_gpu_scan_filter.py -q -x -k "filter" > $o/filter_tests_41.log 2>&1; echo "rc=$?" >> $o/filter_tests_41.log
tail -2 $o/filter_tests_41.log
for rep in 1 2 3; do
  for cfg in 38 41; do
    PIP_FILTER_CFG=$cfg timeout 600 python bench.py --op filter --steps 10 --warmup 3 --no-cpu --no-e2e >> $o/fcfg$cfg.json 2>> $o/fcfg$cfg.err
  done
done
python tools/var_summary.py $o
