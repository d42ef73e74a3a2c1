set -u
o=gpurun_out/rpmid2
mkdir -p $o
for lg in 26 27; do
  for bm in "" 3; do
    PIP_RP_BM=$bm PIP_TIMING=1 timeout 600 python bench.py --op rp --log2n $lg --steps 5 --warmup 2 --no-cpu --no-e2e >> $o/lg${lg}_bm${bm:-d}.json 2>> $o/lg${lg}_bm${bm:-d}.err
  done
  PIP_RP_DBG=2 PIP_TIMING=1 timeout 600 python bench.py --op rp --log2n $lg --steps 5 --warmup 2 --no-cpu --no-e2e >> $o/lg${lg}_bmd_exch.json 2>> $o/lg${lg}_bmd_exch.err
done
python tools/var_summary.py $o
