#!/bin/bash
# Round-end measurement set: bench line, ncu launch list of the bench, full ncu captures of the dominant
# 2D kernel (4 launches of one bench step) and of the 3D kernel (one 512^3 phi_0 call), config sweep.
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 > gpurun_out/b_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_leja2d_tb2 -s 4 -c 4 -o gpurun_out/leja_tb2_full python tools/profile_run.py step 4096 0 > gpurun_out/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_leja3d_smem -s 1 -c 1 -o gpurun_out/leja3d_smem_full python tools/profile_run.py leja3d 512 0 > gpurun_out/ncu3d.log 2>&1
timeout 900 python tools/sweep.py > gpurun_out/sweep.jsonl 2> gpurun_out/sweep.err
ls -la gpurun_out
# summaries (the .ncu-rep files exceed gpurun's 64 MiB return limit)
python tools/ncu_traffic.py gpurun_out/leja_tb2_full.ncu-rep 16,16,14,10 4096 tb2 "ncu --set full --clock-control none, the 4 Leja calls (phi_0..phi_3) of one bench step at 4096^2 (round 1 final, two-step kernel)" > gpurun_out/leja_traffic.json
ncu -i gpurun_out/leja_tb2_full.ncu-rep --page details --csv > gpurun_out/ncu_full_leja_tb2_details.csv 2>/dev/null
ncu -i gpurun_out/leja3d_smem_full.ncu-rep --page details --csv > gpurun_out/ncu_full_leja3d_smem_details.csv 2>/dev/null
ncu -i gpurun_out/leja3d_smem_full.ncu-rep --page raw --csv --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct,launch__registers_per_thread > gpurun_out/ncu_leja3d_smem_raw.csv 2>/dev/null
rm -f gpurun_out/*.ncu-rep
ls -la gpurun_out
