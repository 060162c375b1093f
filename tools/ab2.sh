# A/B of two library builds on the same box: Leja it/s of config 1 (phi_0..phi_3) at several sizes
mkdir -p gpurun_out
: > gpurun_out/ab.txt
for rep in 1 2 3; do
for lib in paper_2310_08344_b200/liblexint_b200_prev.so paper_2310_08344_b200/liblexint_b200.so; do
LX_LIBRARY=$PWD/$lib TAG=$(basename $lib) timeout 120 python tools/ab_n.py ${SIZES:-2048,4096,8192} >> gpurun_out/ab.txt 2>&1
done; done
cat gpurun_out/ab.txt
