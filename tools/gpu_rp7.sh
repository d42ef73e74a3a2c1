set -u
o=gpurun_out/rp7
mkdir -p $o
for c in 1 8; do
PIP_RP_CLUSTER=$c PIP_TIMING=1 timeout 300 python bench.py --op rp0 --steps 5 --warmup 3 --no-cpu --no-e2e > $o/bench_rp0_c$c.json 2> $o/bench_rp0_c$c.err
done
timeout 900 python -m pytest tests/test_gpu_rp_merge.py -q -x -k "reservation_modes" > $o/rp_tests.log 2>&1; echo "rc=$?" >> $o/rp_tests.log
