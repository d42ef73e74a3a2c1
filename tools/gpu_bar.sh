set -u
o=gpurun_out/bar
mkdir -p $o
for op in rp0 rp; do
  PIP_TIMING=1 timeout 600 python bench.py --op $op --steps 5 --warmup 3 --no-cpu --no-e2e > $o/${op}_base.json 2> $o/${op}_base.err
done
rm -rf /tmp/var && cp -r . /tmp/var && cd /tmp/var && PIP_NVCC_EXTRA="-DPIP_BAR_SPIN=1000000" python -m paper_2103_01216_b200._build --force > /dev/null 2>&1
for op in rp0 rp; do
  PIP_TIMING=1 timeout 600 python bench.py --op $op --steps 5 --warmup 3 --no-cpu --no-e2e > $GRAFT_REPO_ROOT/$o/${op}_spin.json 2> $GRAFT_REPO_ROOT/$o/${op}_spin.err
done
