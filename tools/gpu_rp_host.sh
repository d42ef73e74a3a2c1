set -u
o=gpurun_out/rh
mkdir -p $o
timeout 900 python -m pytest tests/test_gpu_rp_host.py tests/test_gpu_rp_merge.py -m gpu -x -q > $o/tests.log 2>&1; echo "rc=$?" >> $o/tests.log
timeout 600 python bench.py --op rp --steps 5 --warmup 3 --no-cpu > $o/bench_rp.json 2> $o/bench_rp.err
PIP_RP_HOST_OVERLAP=0 timeout 600 python bench.py --op rp --steps 3 --warmup 3 --no-cpu > $o/bench_rp_nooverlap.json 2> $o/bench_rp_nooverlap.err
timeout 600 python bench.py --op rp0 --steps 5 --warmup 3 --no-cpu > $o/bench_rp0.json 2> $o/bench_rp0.err
