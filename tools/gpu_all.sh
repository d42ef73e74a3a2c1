set -u
o=gpurun_out/${1:-all}
mkdir -p $o
timeout 2400 python -m pytest tests -m gpu -x -q --durations=15 > $o/gpu_tests.log 2>&1; echo "tests rc=$?" >> $o/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $o/smoke.log 2>&1; echo "smoke rc=$?" >> $o/smoke.log
