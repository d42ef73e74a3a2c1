set -u
o=gpurun_out/wsplit2
mkdir -p $o
for w in "4 4" "5 4" "6 4" "7 4" "8 4" "12 4"; do
  set -- $w
  PIP_RP_WF=$1 PIP_RP_WN=$2 PIP_TIMING=1 timeout 600 python bench.py --op rp --steps 3 --warmup 2 --no-cpu --no-e2e >> $o/w$1_$2.json 2>> $o/w$1_$2.err
done
python tools/var_summary.py $o
