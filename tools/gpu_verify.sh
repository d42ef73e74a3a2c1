set -u
o=gpurun_out/${OUT:-v2}
mkdir -p $o
nvidia-smi > $o/gpu.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $o/gpu_tests.log 2>&1; echo "tests rc=$?" >> $o/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $o/smoke.log 2>&1; echo "smoke rc=$?" >> $o/smoke.log
for op in scan filter merge rp rp0 partition; do
  timeout 600 python bench.py --op $op --steps 5 --warmup 3 > $o/bench_$op.json 2> $o/bench_$op.err
done
timeout 300 python bench.py > $o/bench_default.json 2> $o/bench_default.err
