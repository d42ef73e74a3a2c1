# quicksort leaf-size sweep (PIP_QS_LEAF) at 2^24 and 2^26 words
mkdir -p gpurun_out/qs6
timeout 400 python -m pytest tests/test_gpu_partition.py -m gpu -q -x > gpurun_out/qs6/tests.log 2>&1; echo rc=$? >> gpurun_out/qs6/tests.log
for L in 524288 1048576 2097152 4194304 8388608; do
  PIP_QS_LEAF=$L timeout 300 python tools/bench_extra.py > gpurun_out/qs6/extra_$L.jsonl 2>>gpurun_out/qs6/extra.err
  PIP_QS_LEAF=$L timeout 300 python tools/bench_extra.py --log2n 26 --reps 2 > gpurun_out/qs6/extra26_$L.jsonl 2>>gpurun_out/qs6/extra.err
done
