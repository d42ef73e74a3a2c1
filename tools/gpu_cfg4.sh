set -u
o=gpurun_out/cfg4
mkdir -p $o
for c in 31 32 33 34; do
  PIP_FILTER_CFG=$c timeout 600 python -m pytest tests/test_gpu_scan_filter.py -q -x -k "filter" > $o/filter${c}_tests.log 2>&1; echo "rc=$?" >> $o/filter${c}_tests.log
  PIP_FILTER_CFG=$c timeout 600 python bench.py --op filter --steps 5 --warmup 3 --no-cpu --no-e2e > $o/filter_c$c.json 2> $o/filter_c$c.err
done
timeout 600 python bench.py --op filter --steps 5 --warmup 3 --no-cpu --no-e2e > $o/filter_c17.json 2> $o/filter_c17.err
