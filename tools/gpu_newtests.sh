set -u
o=gpurun_out/nt
mkdir -p $o
timeout 900 python -m pytest tests/test_gpu_contraction.py tests/test_gpu_detres.py -q -x > $o/tests.log 2>&1; echo "rc=$?" >> $o/tests.log
