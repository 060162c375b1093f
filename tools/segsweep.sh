mkdir -p gpurun_out
: > gpurun_out/segsweep.txt
for rep in 1 2; do
LX_TB2_SEG=8 TAG=seg8 timeout 120 python tools/ab_n.py 2048,4096,8192 >> gpurun_out/segsweep.txt 2>&1
for g in "16,32,1" "16,32,2" "24,32,2" "16,48,2" "32,32,1" "16,32,4"; do
LX_TB2_GUIDED=$g TAG=g$g timeout 120 python tools/ab_n.py 2048,4096,8192 >> gpurun_out/segsweep.txt 2>&1
done
done
cat gpurun_out/segsweep.txt
