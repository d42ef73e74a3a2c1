# A/B: variant tree /tmp/varB gets tools/_ab/lookback_old.cuh; alternate runs
set -u
o=gpurun_out/ab2
mkdir -p $o
python -m paper_2103_01216_b200._build > $o/build.log 2>&1
rm -rf /tmp/varB && cp -r . /tmp/varB && cp tools/_ab/lookback_old.cuh /tmp/varB/paper_2103_01216_b200/csrc/lookback.cuh && (cd /tmp/varB && python -m paper_2103_01216_b200._build --force > /dev/null 2>&1)
for rep in 1 2 3; do
  for op in filter scan; do
    timeout 600 python bench.py --op $op --steps 10 --warmup 3 --no-cpu --no-e2e >> $o/new.jsonl 2>> $o/err
    (cd /tmp/varB && timeout 600 python bench.py --op $op --steps 10 --warmup 3 --no-cpu --no-e2e) >> $o/old.jsonl 2>> $o/err
  done
done
true
