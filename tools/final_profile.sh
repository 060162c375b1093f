#!/bin/bash
# Round-end measurement set (run under gpurun from the repo root): bench lines of the BASELINE configs, the
# ncu launch lists of the default bench and of one config-5 step, full ncu captures of the dominant 2D kernel
# (the 4 Leja launches of one bench step) and of config 5's dominant 3D call (vertical phi_1 K = 3), the
# slab-cost tables (2D, 3D), the NCCL self-check and the config sweep (incl. the config-1 dt sweep).
# Summaries land in gpurun_out/ (the .ncu-rep files exceed gpurun's return limit and are deleted).
set -x
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --config 4 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
timeout 600 python bench.py --config 4 --n 8192 --no-cpu > gpurun_out/bench_c4_8192.json 2> gpurun_out/bench_c4_8192.err
timeout 600 python bench.py --config 5 --steps 5 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu --no-exprb > gpurun_out/b_ncu.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -c 300 --csv --log-file gpurun_out/launches_c5.csv \
    python bench.py --config 5 --steps 1 --warmup 3 --no-cpu > gpurun_out/c5_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_leja2d_tb2 -s 8 -c 4 \
    -o gpurun_out/leja_tb2_full python tools/profile_run.py step 4096 0 3 > gpurun_out/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k regex:"tb2<.int.3" -s 1 -c 1 -o gpurun_out/vert3d_full python tools/profile_run.py vert3d 512 1 \
    > gpurun_out/ncu_vert3d.log 2>&1
timeout 600 python tools/slab_cost.py 4096 4096 > gpurun_out/slab_cost.jsonl 2>&1
timeout 600 python tools/slab_cost.py 1024 8192 >> gpurun_out/slab_cost.jsonl 2>&1
timeout 600 python tools/slab_cost.py 64 512 512 > gpurun_out/slab_cost3d.jsonl 2>&1
timeout 600 python tools/nccl_selfcheck.py --time > gpurun_out/nccl_selfcheck.json 2>&1
timeout 1200 python tools/sweep.py > gpurun_out/sweep.jsonl 2> gpurun_out/sweep.err
python tools/ncu_traffic.py gpurun_out/leja_tb2_full.ncu-rep 16,16,14,10 4096 tb2 \
    "ncu --set full --clock-control none, the 4 Leja calls (phi_0..phi_3) of one bench step at 4096^2 (round 2, pipelined two-step kernel)" \
    > gpurun_out/leja_traffic.json
ACC=$(grep -o "accumulators [0-9:]*" gpurun_out/ncu_vert3d.log | awk '{print $2}')
python tools/ncu_traffic.py gpurun_out/vert3d_full.ncu-rep "$ACC" 512 vert3d \
    "ncu --set full --clock-control none, config 5's dominant call: vertical phi_1 {1/2, 2/3, 1} on f(u) dt at 512^3 (k_leja3d_tb2<3>)" \
    > gpurun_out/leja3d_traffic.json
ncu -i gpurun_out/leja_tb2_full.ncu-rep --page details --csv > gpurun_out/ncu_full_leja_tb2_details.csv 2>/dev/null
ncu -i gpurun_out/vert3d_full.ncu-rep --page details --csv > gpurun_out/ncu_full_vert3d_details.csv 2>/dev/null
rm -f gpurun_out/*.ncu-rep
ls -la gpurun_out
