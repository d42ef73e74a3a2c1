set -u
o=gpurun_out/cfg5
mkdir -p $o
timeout 600 python -m pytest tests/test_gpu_scan_filter.py -q -x -k "filter" > $o/filter_tests.log 2>&1; echo "rc=$?" >> $o/filter_tests.log
for i in 1 2; do
timeout 600 python bench.py --op filter --steps 5 --warmup 3 --no-cpu --no-e2e > $o/filter_$i.json 2> $o/filter_$i.err
done
