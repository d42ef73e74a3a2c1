set -u
o=gpurun_out/rpmid3
mkdir -p $o
for lg in 22 24 26 27 28; do
  PIP_TIMING=1 timeout 600 python bench.py --op rp --log2n $lg --steps 5 --warmup 2 --no-cpu --no-e2e >> $o/lg${lg}_bm1.json 2>> $o/lg${lg}_bm1.err
  PIP_RP_DBG=2 PIP_TIMING=1 timeout 600 python bench.py --op rp --log2n $lg --steps 5 --warmup 2 --no-cpu --no-e2e >> $o/lg${lg}_bm1_exch.json 2>> $o/lg${lg}_bm1_exch.err
  PIP_RP_BM=3 PIP_TIMING=1 timeout 600 python bench.py --op rp --log2n $lg --steps 5 --warmup 2 --no-cpu --no-e2e >> $o/lg${lg}_bm3.json 2>> $o/lg${lg}_bm3.err
done
python tools/var_summary.py $o
