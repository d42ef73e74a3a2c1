set -u
o=gpurun_out/rp9
mkdir -p $o
timeout 900 python -m pytest tests/test_gpu_rp_merge.py tests/test_gpu_rp_host.py tests/test_gpu_detres.py tests/test_sharded_abi.py -q -x > $o/rp_tests.log 2>&1; echo "rc=$?" >> $o/rp_tests.log
tail -3 $o/rp_tests.log
bash tools/gpu_var.sh rp9 "m7" --op rp --steps 3 --warmup 2 --no-cpu --no-e2e
for i in 1 2; do PIP_TIMING=1 timeout 600 python bench.py --op rp0 --steps 10 --warmup 3 --no-cpu --no-e2e >> $o/rp0.json 2>> $o/rp0.err; done
cut -c90-200 $o/rp0.json; grep "pip rp" $o/rp0.err | tail -1
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x -k "rp or perm" > $o/full_tests.log 2>&1; echo "rc=$?" >> $o/full_tests.log
tail -3 $o/full_tests.log
