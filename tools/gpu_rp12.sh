set -u
o=gpurun_out/rp12
mkdir -p $o
for rep in 1 2; do
for ipt in 1 2 3 4; do
  PIP_RP_IPT=$ipt PIP_TIMING=1 timeout 600 python bench.py --op rp0 --steps 20 --warmup 5 --no-cpu --no-e2e >> $o/ipt$ipt.json 2>> $o/ipt$ipt.err
done
done
python tools/var_summary.py $o
