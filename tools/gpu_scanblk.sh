set -u
o=gpurun_out/scanblk
mkdir -p $o
PIP_SCAN_CFG=20 timeout 900 python -m pytest tests/test_gpu_scan_filter.py tests/test_gpu_scan_filter_host.py -q -x -k "scan" > $o/tests.log 2>&1; echo "rc=$?" >> $o/tests.log
for c in 17 20 17 20; do
  PIP_SCAN_CFG=$c timeout 600 python bench.py --op scan --steps 5 --warmup 3 --no-cpu --no-e2e >> $o/scan5_c$c.jsonl 2>> $o/err.log
done
for c in 17 20; do
  PIP_SCAN_CFG=$c timeout 600 python bench.py --op scan --steps 20 --warmup 3 --no-cpu --no-e2e > $o/scan20_c$c.json 2>> $o/err.log
done
