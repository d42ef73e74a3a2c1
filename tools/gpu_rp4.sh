set -u
o=gpurun_out/rp4
mkdir -p $o
timeout 900 python -m pytest tests/test_gpu_rp_merge.py tests/test_gpu_rp_host.py tests/test_gpu_boundary.py tests/test_gpu_detres.py -q -x -k "rp or boundary or detres" > $o/rp_tests.log 2>&1; echo "rc=$?" >> $o/rp_tests.log
timeout 300 python bench.py --op rp0 --steps 20 --warmup 3 --no-cpu > $o/bench_rp0.json 2> $o/bench_rp0.err
PIP_RP_CLUSTER=0 timeout 300 python bench.py --op rp0 --steps 20 --warmup 3 --no-cpu --no-e2e > $o/bench_rp0_nocluster.json 2> $o/bench_rp0_nocluster.err
for cfg in "PIP_RP_BM=2" "PIP_RP_BM=2 PIP_RP_DBG=1" "PIP_RP_BM=3 PIP_RP_TLOAD=4" "PIP_RP_BM=3 PIP_RP_DBG=1" "PIP_RP_BM=2 PIP_RP_TLOAD=8"; do
  tag=$(echo $cfg | tr ' =' '__')
  env $cfg PIP_TIMING=1 timeout 600 python bench.py --op rp --steps 2 --warmup 1 --no-e2e --no-cpu > $o/rp_$tag.json 2> $o/rp_$tag.err
done
PIP_RP_BM=2 timeout 600 python bench.py --op rp --steps 1 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1 && \
PIP_RP_BM=2 ncu --set full --clock-control none --import-source on -k regex:rp_kernel -c 1 -o $o/rp_full python bench.py --op rp --steps 1 --warmup 1 --no-e2e --no-cpu > $o/rp_full.log 2>&1
