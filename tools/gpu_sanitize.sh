set -u
o=gpurun_out/san
mkdir -p $o
timeout 300 python tools/sanitize_smoke.py > $o/plain.log 2>&1; echo "rc=$?" >> $o/plain.log
tail -2 $o/plain.log
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_smoke.py > $o/$tool.log 2>&1; echo "rc=$?" >> $o/$tool.log
  echo "== $tool"; tail -6 $o/$tool.log
done
