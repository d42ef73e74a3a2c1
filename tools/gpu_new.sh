set -u
o=gpurun_out/${OUT:-new2}
mkdir -p $o
timeout 900 python -m pytest tests/test_distributed.py tests/test_gpu_boundary.py -q -x -m gpu > $o/dist_tests.log 2>&1; echo "rc=$?" >> $o/dist_tests.log
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -q -rs --durations=0 > $o/fullsize.log 2>&1; echo "rc=$?" >> $o/fullsize.log
for op in filter merge rp; do
  timeout 900 python bench.py --op $op --steps 5 --warmup 3 > $o/bench_$op.json 2> $o/bench_$op.err
done
