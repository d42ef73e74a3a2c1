set -u
PIP_RP_DBG=2 bash tools/gpu_var.sh occ4 "m4s m5s m6s m8s" --op rp --steps 3 --warmup 2 --no-cpu --no-e2e
o=gpurun_out/occ4
cp build/var/libpip_m6s.so paper_2103_01216_b200/libpip.so
PIP_RP_PERSM=6 timeout 900 python -m pytest tests/test_gpu_rp_merge.py tests/test_gpu_rp_host.py tests/test_gpu_detres.py -q -x -k "rp or detres" > $o/rp_tests_m6s.log 2>&1; echo "rc=$?" >> $o/rp_tests_m6s.log
tail -3 $o/rp_tests_m6s.log
