set -u
o=gpurun_out/lbs3
mkdir -p $o
for lg in 30 31 32; do
  PIP_SCAN_CFG=25 PIP_LB_STRIDE=1 timeout 150 python bench.py --op scan --log2n $lg --steps 2 --warmup 1 --no-cpu --no-e2e >> $o/c25_st1_lg$lg.json 2>> $o/c25_st1_lg$lg.err; echo "lg$lg rc=$?"
  PIP_SCAN_CFG=29 PIP_LB_STRIDE=1 timeout 150 python bench.py --op scan --log2n $lg --steps 2 --warmup 1 --no-cpu --no-e2e >> $o/c29_st1_lg$lg.json 2>> $o/c29_st1_lg$lg.err; echo "lg$lg static rc=$?"
done
python tools/var_summary.py $o
