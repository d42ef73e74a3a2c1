set -u
o=gpurun_out/soak2
mkdir -p $o
run() { tag=$1; shift; env "$@" timeout 400 python tools/scan_soak.py 32 $REPS > $o/$tag.log 2>&1; echo "rc=$?" >> $o/$tag.log; echo "== $tag"; tail -4 $o/$tag.log; }
REPS=30 run c29_st1 PIP_SCAN_CFG=29 PIP_LB_STRIDE=1
REPS=100 run c29_def PIP_SCAN_CFG=29
REPS=30 run c21_st1 PIP_SCAN_CFG=21 PIP_LB_STRIDE=1
REPS=60 run c25_st2 PIP_SCAN_CFG=25 PIP_LB_STRIDE=2
REPS=30 run c25_st1_again PIP_SCAN_CFG=25 PIP_LB_STRIDE=1
