set -u
o=gpurun_out/rp0m
mkdir -p $o
for bm in 0 1 2 3; do
  PIP_RP_BM=$bm PIP_TIMING=1 timeout 300 python bench.py --op rp0 --steps 10 --warmup 3 --no-cpu --no-e2e > $o/rp0_bm$bm.json 2> $o/rp0_bm$bm.err
done
for ipt in 2 4; do
  PIP_RP_IPT=$ipt PIP_TIMING=1 timeout 300 python bench.py --op rp0 --steps 10 --warmup 3 --no-cpu --no-e2e > $o/rp0_ipt$ipt.json 2> $o/rp0_ipt$ipt.err
done
