set -u
o=gpurun_out/multi
mkdir -p $o
for op in scan filter merge; do
  for ws in 2 3; do
    PIP_ONE_GPU=1 PIP_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$ws \
      --master-addr 127.0.0.1 --master-port $((29500 + ws)) bench.py --gpus $ws --op $op --log2n 24 \
      --steps 2 --warmup 1 --no-e2e --no-cpu > $o/${op}_ws$ws.json 2> $o/${op}_ws$ws.err
    echo "rc=$?" >> $o/${op}_ws$ws.err
  done
done
timeout 900 python -m pytest tests/test_gpu_move.py -q > $o/move_tests.log 2>&1; echo "rc=$?" >> $o/move_tests.log
