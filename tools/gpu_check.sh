#!/bin/bash
# One GPU session: parity tests, bench (default + one-step kernel), ncu launch list + full capture of the top kernel.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
LX_TBLOCK=1 timeout 600 python bench.py > gpurun_out/bench_tb1.json 2> gpurun_out/bench_tb1.err
if [ "${NCU:-1}" = 1 ]; then
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 > gpurun_out/b_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_leja2d_tb2 -s 4 -c 4 -o gpurun_out/leja_tb2_full python tools/profile_run.py step 4096 0 > gpurun_out/ncu_full.log 2>&1
fi
