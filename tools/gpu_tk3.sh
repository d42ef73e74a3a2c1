set -u
o=gpurun_out/tk4
mkdir -p $o
for rep in 1 2; do
  for cfg in 21 22 25 26 27; do
    PIP_SCAN_CFG=$cfg timeout 600 python bench.py --op scan --steps 10 --warmup 3 --no-cpu --no-e2e >> $o/cfg$cfg.json 2>> $o/cfg$cfg.err
  done
done
python tools/var_summary.py $o
