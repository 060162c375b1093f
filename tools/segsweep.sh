mkdir -p gpurun_out
: > gpurun_out/segsweep.txt
for rep in 1 2; do
for sc in fixed balanced; do
LX_TB2_SCHED=$sc TAG=$sc timeout 120 python tools/ab_n.py 2048,3072,4096,6144,8192 >> gpurun_out/segsweep.txt 2>&1
done; done
cat gpurun_out/segsweep.txt
