set -u
o=gpurun_out/rp6
mkdir -p $o
PIP_TIMING=1 timeout 300 python bench.py --op rp0 --steps 5 --warmup 3 --no-cpu --no-e2e > $o/bench_rp0.json 2> $o/bench_rp0.err
PIP_RP_CLUSTER=0 PIP_TIMING=1 timeout 300 python bench.py --op rp0 --steps 5 --warmup 3 --no-cpu --no-e2e > $o/bench_rp0_grid.json 2> $o/bench_rp0_grid.err
timeout 300 python bench.py --op rp0 --steps 5 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $o/launches_rp0.csv python bench.py --op rp0 --steps 5 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
