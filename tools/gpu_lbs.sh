set -u
o=gpurun_out/lbs
mkdir -p $o
for rep in 1 2; do
for st in 1 2 4 8; do
  PIP_LB_STRIDE=$st timeout 600 python bench.py --op scan --steps 10 --warmup 3 --no-cpu --no-e2e >> $o/scan_st$st.json 2>> $o/scan_st$st.err
  PIP_LB_STRIDE=$st timeout 600 python bench.py --op filter --steps 10 --warmup 3 --no-cpu --no-e2e >> $o/filter_st$st.json 2>> $o/filter_st$st.err
done
done
python tools/var_summary.py $o
