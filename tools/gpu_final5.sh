set -u
o=gpurun_out/final5
mkdir -p $o
nvidia-smi > $o/gpu.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q --durations=10 > $o/gpu_tests.log 2>&1; echo "tests rc=$?" >> $o/gpu_tests.log
tail -3 $o/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $o/smoke.log 2>&1; echo "smoke rc=$?" >> $o/smoke.log
tail -2 $o/smoke.log
for rep in 1 2; do for cfg in 38 40; do
  PIP_FILTER_CFG=$cfg timeout 600 python bench.py --op filter --steps 10 --warmup 3 --no-cpu --no-e2e >> $o/fcfg$cfg.json 2>> $o/fcfg$cfg.err
done; done
python tools/var_summary.py $o
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $o/ref_default.json 2> $o/ref_default.err
timeout 600 python bench.py --steps 20 --warmup 5 > $o/bench_default.json 2> $o/bench_default.err
for op in scan filter merge rp rp0 partition; do
  timeout 900 python bench.py --op $op --steps 5 --warmup 3 > $o/bench_$op.json 2> $o/bench_$op.err
done
cat $o/bench_*.json | cut -c1-330
