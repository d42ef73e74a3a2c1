set -u
o=gpurun_out/rp3
mkdir -p $o
timeout 900 python -m pytest tests/test_distributed.py tests/test_gpu_boundary.py -q -x -m gpu > $o/dist_tests.log 2>&1; echo "rc=$?" >> $o/dist_tests.log
timeout 900 python -m pytest tests/test_gpu_rp_merge.py -q -x -k "reservation_modes or rp" > $o/rp_tests.log 2>&1; echo "rc=$?" >> $o/rp_tests.log
for bm in 2 3; do
  PIP_RP_BM=$bm PIP_TIMING=1 timeout 600 python bench.py --op rp --steps 3 --warmup 2 --no-e2e --no-cpu > $o/bench_rp_bm$bm.json 2> $o/bench_rp_bm$bm.err
done
for f in 27 29; do
  PIP_RP_FOLD_LOG2=$f timeout 600 python bench.py --op rp --steps 3 --warmup 2 --no-e2e --no-cpu > $o/bench_rp_f$f.json 2> $o/bench_rp_f$f.err
done
timeout 600 python bench.py --op rp --steps 3 --warmup 2 --no-e2e --no-cpu > $o/plain_rp.json 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:rp_kernel -c 3 --csv --log-file $o/rp_ncu.csv python bench.py --op rp --steps 1 --warmup 1 --no-e2e --no-cpu > $o/rp_ncu.log 2>&1
