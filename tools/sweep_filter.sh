# filter pipeline-shape sweep: parity tests then bench at 2^32 for each config
set -u
o=gpurun_out/sf
mkdir -p $o
for c in ${CFGS:-23 24 25 17}; do
  PIP_FILTER_CFG=$c timeout 600 python -m pytest tests/test_gpu_scan_filter.py -m gpu -x -q -k "filter" > $o/tests_$c.log 2>&1; echo "rc=$?" >> $o/tests_$c.log
  PIP_FILTER_CFG=$c timeout 300 python bench.py --op filter --steps 5 --warmup 3 --no-cpu --no-e2e > $o/bench_$c.json 2> $o/bench_$c.err
done
