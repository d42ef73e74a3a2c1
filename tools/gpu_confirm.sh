set -u
o=gpurun_out/${1:-confirm}
mkdir -p $o
nvidia-smi > $o/gpu.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q --durations=15 > $o/gpu_tests.log 2>&1; echo "tests rc=$?" >> $o/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $o/smoke.log 2>&1; echo "smoke rc=$?" >> $o/smoke.log
timeout 600 python bench.py > $o/bench_default.json 2> $o/bench_default.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $o/ref_default.json 2> $o/ref_default.err
for op in filter merge rp rp0; do
  timeout 900 python bench.py --op $op --steps 5 --warmup 3 > $o/bench_$op.json 2> $o/bench_$op.err
done
tail -3 $o/gpu_tests.log; cat $o/smoke.log | tail -2; cat $o/bench_*.json | cut -c1-400
