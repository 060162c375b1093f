# A/B of 3D tile variants: 512^3 phi_0 call + EPIRK4s3A step (tools/sweep.py config 4)
mkdir -p gpurun_out; : > gpurun_out/ab3d.txt
for rep in 1 2; do for lib in liblexint_b200.so liblexint_b200_rt4.so; do
echo $lib >> gpurun_out/ab3d.txt
LX_LIBRARY=$PWD/paper_2310_08344_b200/$lib timeout 300 python tools/sweep.py --only 4 >> gpurun_out/ab3d.txt 2>&1
done; done
LX_LIBRARY=$PWD/paper_2310_08344_b200/liblexint_b200_rt4.so timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_slab.py -q -x -k "3d or 3D" >> gpurun_out/ab3d.txt 2>&1
cat gpurun_out/ab3d.txt
