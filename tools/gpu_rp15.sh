set -u
o=gpurun_out/rp15
mkdir -p $o
timeout 900 python -m pytest tests/test_gpu_rp_merge.py tests/test_gpu_rp_host.py tests/test_gpu_detres.py -q -x > $o/rp_tests.log 2>&1; echo "rc=$?" >> $o/rp_tests.log
tail -2 $o/rp_tests.log
for rep in 1 2; do
PIP_TIMING=1 timeout 600 python bench.py --op rp0 --steps 20 --warmup 5 --no-cpu --no-e2e >> $o/cl1024.json 2>> $o/cl1024.err
PIP_RP_CL1=0 PIP_TIMING=1 timeout 600 python bench.py --op rp0 --steps 20 --warmup 5 --no-cpu --no-e2e >> $o/grid.json 2>> $o/grid.err
cp paper_2103_01216_b200/libpip.so /tmp/libpip_base.so; cp build/var/libpip_clt512.so paper_2103_01216_b200/libpip.so
PIP_TIMING=1 timeout 600 python bench.py --op rp0 --steps 20 --warmup 5 --no-cpu --no-e2e >> $o/cl512.json 2>> $o/cl512.err
cp /tmp/libpip_base.so paper_2103_01216_b200/libpip.so
done
python tools/var_summary.py $o
