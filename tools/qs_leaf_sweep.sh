mkdir -p gpurun_out/qs4
for L in 65536 131072 262144 524288 1048576; do
  PIP_QS_LEAF=$L timeout 300 python tools/bench_extra.py > gpurun_out/qs4/extra_$L.jsonl 2>>gpurun_out/qs4/extra.err
done
PIP_QS_LEAF=262144 timeout 400 python -m pytest tests/test_gpu_partition.py -m gpu -q -x -k "quicksort or sort_segments" > gpurun_out/qs4/tests.log 2>&1; echo rc=$? >> gpurun_out/qs4/tests.log
