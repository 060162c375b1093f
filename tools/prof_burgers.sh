#!/bin/bash
# Burgers phi_1 (flux-form Jacobian) measurement: full ncu capture of one warm Leja call at 4096^2.
set -x
mkdir -p gpurun_out
python tools/prof_burgers.py > gpurun_out/burgers_plain.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_leja2d -s 1 -c 1 \
    -o gpurun_out/burgers_full python tools/prof_burgers.py > gpurun_out/ncu_burgers.log 2>&1
ncu -i gpurun_out/burgers_full.ncu-rep --page details --csv > gpurun_out/ncu_full_burgers_details.csv 2>/dev/null
ncu -i gpurun_out/burgers_full.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu_burgers_sass.csv 2>/dev/null
ncu -i gpurun_out/burgers_full.ncu-rep --page raw --csv > gpurun_out/ncu_burgers_raw.csv 2>/dev/null
rm -f gpurun_out/*.ncu-rep
