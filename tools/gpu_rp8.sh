set -u
o=gpurun_out/rp8
mkdir -p $o
PIP_TIMING=1 timeout 600 python bench.py --op rp --steps 3 --warmup 2 --no-cpu --no-e2e > $o/rp.json 2> $o/rp.err
PIP_TIMING=1 timeout 600 python bench.py --op rp0 --steps 10 --warmup 3 --no-cpu --no-e2e > $o/rp0.json 2> $o/rp0.err
timeout 900 python -m pytest tests/test_gpu_rp_merge.py tests/test_gpu_rp_host.py tests/test_gpu_detres.py -q -x -k "rp or detres" > $o/rp_tests.log 2>&1; echo "rc=$?" >> $o/rp_tests.log
