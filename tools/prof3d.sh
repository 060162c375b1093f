#!/bin/bash
# 3D (config 5) measurement set, run under gpurun from the repo root: launch list of one warm EPIRK4s3A step
# at 512^3, a full ncu capture of the step's dominant call (vertical phi_1 {1/2, 2/3, 1}, K = 3) with the
# per-SASS-instruction source page, and its traffic summary (profiles/leja3d_traffic.json).
set -x
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -c 300 --csv --log-file gpurun_out/launches_c5.csv \
    python bench.py --config 5 --steps 1 --warmup 3 --no-cpu > gpurun_out/c5_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"tb2<.int.3" -s 1 -c 1 \
    -o gpurun_out/vert3d_full python tools/profile_run.py vert3d 512 1 > gpurun_out/ncu_vert3d.log 2>&1
ACC=$(grep -o "accumulators [0-9:]*" gpurun_out/ncu_vert3d.log | awk '{print $2}')
python tools/ncu_traffic.py gpurun_out/vert3d_full.ncu-rep "$ACC" 512 vert3d \
    "ncu --set full --clock-control none, config 5's dominant call: vertical phi_1 {1/2, 2/3, 1} on f(u) dt at 512^3 (k_leja3d_tb2<3>)" \
    > gpurun_out/leja3d_traffic.json
ncu -i gpurun_out/vert3d_full.ncu-rep --page details --csv > gpurun_out/ncu_full_vert3d_details.csv 2>/dev/null
ncu -i gpurun_out/vert3d_full.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu_vert3d_sass.csv 2>/dev/null
rm -f gpurun_out/*.ncu-rep
ls -la gpurun_out
