set -u
o=gpurun_out/tree2
mkdir -p $o
for i in 1 2; do
timeout 600 python tools/bench_extra.py --only tree --log2n 24 --reps 5 > $o/tree24_$i.jsonl 2> $o/tree24_$i.err
done
