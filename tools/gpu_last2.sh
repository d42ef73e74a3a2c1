set -u
o=gpurun_out/last2
mkdir -p $o
PIP_LB_STRIDE=1 timeout 400 python tools/filter_soak.py 32 40 > $o/filter_soak_st1.log 2>&1; echo "rc=$?" >> $o/filter_soak_st1.log; tail -2 $o/filter_soak_st1.log
timeout 400 python tools/filter_soak.py 32 150 > $o/filter_soak_default.log 2>&1; echo "rc=$?" >> $o/filter_soak_default.log; tail -2 $o/filter_soak_default.log
timeout 2400 python -m pytest tests -m gpu -x -q > $o/gpu_tests.log 2>&1; echo "tests rc=$?" >> $o/gpu_tests.log
tail -3 $o/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $o/smoke.log 2>&1; echo "smoke rc=$?" >> $o/smoke.log
tail -2 $o/smoke.log
timeout 600 python bench.py --steps 20 --warmup 5 > $o/bench_default.json 2> $o/bench_default.err
cut -c1-300 $o/bench_default.json
