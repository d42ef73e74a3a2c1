set -u
o=gpurun_out/tree
mkdir -p $o
timeout 900 python -m pytest tests/test_gpu_contraction.py -q -x > $o/tests.log 2>&1; echo "rc=$?" >> $o/tests.log
timeout 600 python tools/bench_extra.py --only tree --log2n 20 > $o/tree20.jsonl 2> $o/tree20.err
timeout 600 python tools/bench_extra.py --only tree --log2n 24 > $o/tree24.jsonl 2> $o/tree24.err
