set -u
o=gpurun_out/soak
mkdir -p $o
PIP_LB_STRIDE=1 timeout 300 python tools/scan_soak.py 32 30 > $o/st1.log 2>&1; echo "rc=$?" >> $o/st1.log; tail -5 $o/st1.log
timeout 300 python tools/scan_soak.py 32 200 > $o/default.log 2>&1; echo "rc=$?" >> $o/default.log; tail -3 $o/default.log
PIP_SCAN_CFG=17 PIP_LB_STRIDE=1 timeout 300 python tools/scan_soak.py 32 30 > $o/c17_st1.log 2>&1; echo "rc=$?" >> $o/c17_st1.log; tail -3 $o/c17_st1.log
