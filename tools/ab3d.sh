# A/B of the 3D Leja kernels (LX_3D_KERNEL=tile|smem): 512^3 phi_0 + EPIRK4s3A step, then parity
mkdir -p gpurun_out; : > gpurun_out/ab3d.txt
for rep in 1 2; do for k in tile smem; do
echo $k >> gpurun_out/ab3d.txt
LX_3D_KERNEL=$k timeout 300 python tools/sweep.py --only 4 >> gpurun_out/ab3d.txt 2>&1
done; done
LX_3D_KERNEL=smem timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -k "3d or 3D or 512" >> gpurun_out/ab3d.txt 2>&1
cat gpurun_out/ab3d.txt | cut -c1-330
