set -u
o=gpurun_out/re
mkdir -p $o
for i in 1 2; do
  timeout 600 python bench.py --op rp --steps 3 --warmup 3 --no-cpu > $o/ov0_$i.json 2>/dev/null
  PIP_RP_POLL_US=50 timeout 600 python bench.py --op rp --steps 3 --warmup 3 --no-cpu > $o/ov50_$i.json 2>/dev/null
  PIP_RP_HOST_OVERLAP=0 timeout 600 python bench.py --op rp --steps 3 --warmup 3 --no-cpu > $o/off_$i.json 2>/dev/null
done
