set -u
o=gpurun_out/ph
mkdir -p $o
timeout 900 python -m pytest tests/test_gpu_partition_host.py tests/test_gpu_partition.py -m gpu -x -q > $o/tests.log 2>&1; echo "rc=$?" >> $o/tests.log
timeout 600 python bench.py --op partition --steps 5 --warmup 3 --no-cpu > $o/bench_partition.json 2> $o/bench_partition.err
PIP_PARTITION_HOST_INPLACE=1 timeout 600 python bench.py --op partition --steps 3 --warmup 3 --no-cpu > $o/bench_partition_inplace.json 2> $o/bench_partition_inplace.err
