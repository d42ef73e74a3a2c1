set -u
o=gpurun_out/rp5
mkdir -p $o
PIP_TIMING=1 timeout 300 python bench.py --op rp0 --steps 20 --warmup 3 --no-cpu --no-e2e > $o/bench_rp0.json 2> $o/bench_rp0.err
timeout 900 python -m pytest tests/test_gpu_rp_merge.py tests/test_gpu_rp_host.py tests/test_gpu_detres.py -q -x -k "rp or detres" > $o/rp_tests.log 2>&1; echo "rc=$?" >> $o/rp_tests.log
for cfg in "PIP_RP_BM=2 PIP_RP_LF=0" "PIP_RP_BM=2" "PIP_RP_BM=2 PIP_RP_FMB=2" "PIP_RP_BM=3" "PIP_RP_BM=3 PIP_RP_FMB=2" "PIP_RP_BM=3 PIP_RP_FMB=2 PIP_RP_DBG=1"; do
  tag=$(echo $cfg | tr ' =' '__')
  env $cfg PIP_TIMING=1 timeout 600 python bench.py --op rp --steps 2 --warmup 1 --no-e2e --no-cpu > $o/rp_$tag.json 2> $o/rp_$tag.err
done
