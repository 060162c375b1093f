# A/B of 3D kernel builds (LX_LIBRARY): 512^3 phi_0 + EPIRK4s3A step
mkdir -p gpurun_out; : > gpurun_out/ab3d.txt
for rep in 1 2; do for lib in "$@"; do
echo $lib >> gpurun_out/ab3d.txt
LX_LIBRARY=$PWD/paper_2310_08344_b200/$lib timeout 300 python tools/sweep.py --only 4 | cut -c60-330 >> gpurun_out/ab3d.txt 2>&1
done; done
cat gpurun_out/ab3d.txt
