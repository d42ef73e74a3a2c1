set -u
o=gpurun_out/${OUT:-new}
mkdir -p $o
free -g > $o/free.txt; nproc >> $o/free.txt
timeout 900 python -m pytest tests/test_gpu_boundary.py tests/test_gpu_detres.py tests/test_gpu_scan_filter_host.py -q -x > $o/new_tests.log 2>&1; echo "rc=$?" >> $o/new_tests.log
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -q -rs --durations=0 > $o/fullsize.log 2>&1; echo "rc=$?" >> $o/fullsize.log
