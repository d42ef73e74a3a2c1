set -u
o=gpurun_out/lbs2
mkdir -p $o
for cfg in 17 21 25 29; do
for st in 1 2; do
  PIP_SCAN_CFG=$cfg PIP_LB_STRIDE=$st timeout 300 python bench.py --op scan --log2n 28 --steps 3 --warmup 3 --no-cpu --no-e2e >> $o/c${cfg}_st$st.json 2>> $o/c${cfg}_st$st.err
done
done
python tools/var_summary.py $o
