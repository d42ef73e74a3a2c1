set -u
o=gpurun_out/mh
mkdir -p $o
timeout 900 python -m pytest tests/test_gpu_merge_host.py tests/test_gpu_rp_merge.py -m gpu -x -q > $o/tests.log 2>&1; echo "rc=$?" >> $o/tests.log
timeout 600 python bench.py --op merge --steps 5 --warmup 3 --no-cpu > $o/bench_merge.json 2> $o/bench_merge.err
PIP_MERGE_HOST_INPLACE=1 timeout 600 python bench.py --op merge --steps 3 --warmup 3 --no-cpu > $o/bench_merge_inplace.json 2> $o/bench_merge_inplace.err
PIP_HOST_CHUNK_LOG2=23 timeout 600 python bench.py --op merge --steps 3 --warmup 3 --no-cpu > $o/bench_merge_c23.json 2> $o/bench_merge_c23.err
PIP_HOST_CHUNK_LOG2=22 PIP_HOST_NBUF=6 timeout 600 python bench.py --op merge --steps 3 --warmup 3 --no-cpu > $o/bench_merge_c22.json 2> $o/bench_merge_c22.err
