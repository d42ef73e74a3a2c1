# run a bench command against prebuilt library variants build/var/libpip_<tag>.so
# usage: gpu_var.sh <outdir> "<tags>" <bench args...>
set -u
o=gpurun_out/$1; tags=$2; shift 2
mkdir -p $o
cp paper_2103_01216_b200/libpip.so /tmp/libpip_base.so
for rep in 1 2; do
for t in base $tags; do
  if [ $t = base ]; then cp /tmp/libpip_base.so paper_2103_01216_b200/libpip.so; else cp build/var/libpip_$t.so paper_2103_01216_b200/libpip.so; fi
  persm=; case $t in m[0-9]*) persm=${t:1:1};; esac
  PIP_RP_PERSM=$persm PIP_TIMING=1 timeout 600 python bench.py "$@" >> $o/$t.json 2>> $o/$t.err
done
done
cp /tmp/libpip_base.so paper_2103_01216_b200/libpip.so
for t in base $tags; do echo $t; cut -c90-220 $o/$t.json; grep -h "pip rp" $o/$t.err | tail -2; done
