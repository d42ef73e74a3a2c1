set -u
o=gpurun_out/wait
mkdir -p $o
for v in 0 200 1000 5000; do
  rm -rf /tmp/var && cp -r . /tmp/var && (cd /tmp/var && PIP_NVCC_EXTRA="-DPIP_WAIT_NS=$v" python -m paper_2103_01216_b200._build --force > /dev/null 2>&1)
  (cd /tmp/var && for op in filter scan; do timeout 600 python bench.py --op $op --steps 5 --warmup 3 --no-cpu --no-e2e; done) > $o/w$v.jsonl 2> $o/w$v.err
done
(cd /tmp/var && timeout 900 python -m pytest tests/test_gpu_scan_filter.py -q -x) > $o/tests_w5000.log 2>&1; echo "rc=$?" >> $o/tests_w5000.log
