set -u
o=gpurun_out/tk6
mkdir -p $o
for rep in 1 2; do
  for cfg in 17 36 37; do
    PIP_FILTER_CFG=$cfg timeout 600 python bench.py --op filter --steps 10 --warmup 3 --no-cpu --no-e2e >> $o/fcfg$cfg.json 2>> $o/fcfg$cfg.err
  done
done
python tools/var_summary.py $o
