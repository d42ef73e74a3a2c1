set -u
o=gpurun_out/exch
mkdir -p $o
timeout 300 python tools/rmw_modes.py > $o/rmw_modes.jsonl 2> $o/rmw_modes.err
for d in 0 2 0 2; do
  PIP_RP_DBG=$d PIP_TIMING=1 timeout 600 python bench.py --op rp --steps 3 --warmup 2 --no-cpu --no-e2e >> $o/rp_dbg$d.json 2>> $o/rp_dbg$d.err
  PIP_RP_DBG=$d timeout 600 python bench.py --op rp0 --steps 10 --warmup 3 --no-cpu --no-e2e >> $o/rp0_dbg$d.json 2>> $o/rp0_dbg$d.err
done
cat $o/rmw_modes.jsonl; for d in 0 2; do cut -c1-200 $o/rp_dbg$d.json; grep -h "commit" $o/rp_dbg$d.err | tail -2; cut -c1-200 $o/rp0_dbg$d.json; done
