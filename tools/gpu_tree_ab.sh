set -u
o=gpurun_out/treeab
mkdir -p $o
rm -rf /tmp/var && cp -r . /tmp/var && cp tools/_tree_old.cu.txt /tmp/var/paper_2103_01216_b200/csrc/tree.cu && (cd /tmp/var && python -m paper_2103_01216_b200._build --force > /dev/null 2>&1)
for i in 1 2 3; do
  timeout 600 python tools/bench_extra.py --only tree --log2n 24 --reps 5 > $o/new_$i.jsonl 2>&1
  (cd /tmp/var && timeout 600 python tools/bench_extra.py --only tree --log2n 24 --reps 5) > $o/old_$i.jsonl 2>&1
done
