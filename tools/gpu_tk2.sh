set -u
o=gpurun_out/tk2
mkdir -p $o
PIP_FILTER_CFG=35 timeout 900 python -m pytest tests/test_gpu_scan_filter.py -q -x -k "filter" > $o/filter_tests.log 2>&1; echo "rc=$?" >> $o/filter_tests.log
tail -2 $o/filter_tests.log
for rep in 1 2 3; do
  for cfg in 17 35; do
    PIP_FILTER_CFG=$cfg timeout 600 python bench.py --op filter --steps 10 --warmup 3 --no-cpu --no-e2e >> $o/fcfg$cfg.json 2>> $o/fcfg$cfg.err
  done
done
for cfg in 17 21; do
  PIP_SCAN_CFG=$cfg timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e >> $o/s20_cfg$cfg.json 2>> $o/s20_cfg$cfg.err
done
python tools/var_summary.py $o
