set -u
o=gpurun_out/rp11
mkdir -p $o
cp paper_2103_01216_b200/libpip.so /tmp/libpip_base.so
for rep in 1 2 3; do
for t in base small1; do
  if [ $t = base ]; then cp /tmp/libpip_base.so paper_2103_01216_b200/libpip.so; else cp build/var/libpip_$t.so paper_2103_01216_b200/libpip.so; fi
  PIP_TIMING=1 timeout 600 python bench.py --op rp0 --steps 20 --warmup 5 --no-cpu --no-e2e >> $o/$t.json 2>> $o/$t.err
done
done
python tools/var_summary.py $o
cp build/var/libpip_small1.so paper_2103_01216_b200/libpip.so
timeout 900 python -m pytest tests/test_gpu_rp_merge.py tests/test_gpu_rp_host.py -q -x > $o/rp_tests_small1.log 2>&1; echo "rc=$?" >> $o/rp_tests_small1.log
tail -2 $o/rp_tests_small1.log
cp /tmp/libpip_base.so paper_2103_01216_b200/libpip.so
