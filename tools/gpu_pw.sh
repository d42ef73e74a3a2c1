# 20-step default runs (the driver's command) alternating library variants on one box
set -u
o=gpurun_out/pw
mkdir -p $o
cp paper_2103_01216_b200/libpip.so /tmp/libpip_base.so
for rep in 1 2 3; do
for t in base w1000; do
  if [ $t = base ]; then cp /tmp/libpip_base.so paper_2103_01216_b200/libpip.so; else cp build/var/libpip_$t.so paper_2103_01216_b200/libpip.so; fi
  timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e >> $o/$t.json 2>> $o/$t.err
  timeout 600 python bench.py --op filter --steps 20 --warmup 5 --no-cpu --no-e2e >> $o/f_$t.json 2>> $o/f_$t.err
done
done
cp /tmp/libpip_base.so paper_2103_01216_b200/libpip.so
python tools/var_summary.py $o
python - <<'PY'
import json,glob
for f in sorted(glob.glob('gpurun_out/pw/*.json')):
    for l in open(f):
        d=json.loads(l); print(f, round(d['ms_per_step'],3), d['clocks'])
PY
