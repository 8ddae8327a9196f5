#!/bin/bash
# c5 matvec pass pairs: launch list, then one full capture (source page) of the last apply's two kernels
mkdir -p gpurun_out
python tools/prof_c5mv.py > gpurun_out/c5mv_plain.log 2>&1 || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"ks_pair" --csv \
    --log-file gpurun_out/c5mv_launches.csv python tools/prof_c5mv.py > /dev/null 2>&1
nmv=$(grep -c "ks_pair" gpurun_out/c5mv_launches.csv)
skip=$((nmv - 2))
timeout 1200 ncu -f --set full --clock-control none --import-source on -k regex:"ks_pair" -s $skip -c 2 \
    -o /tmp/prof_c5mv python tools/prof_c5mv.py > gpurun_out/ncu_c5mv.log 2>&1
python tools/ncu_summary.py /tmp/prof_c5mv.ncu-rep gpurun_out/ncu_c5mv_summary.csv >> gpurun_out/ncu_c5mv.log 2>&1
ncu -i /tmp/prof_c5mv.ncu-rep --page source --csv > gpurun_out/ncu_c5mv_source.csv 2>/dev/null
ncu -i /tmp/prof_c5mv.ncu-rep --page details > gpurun_out/ncu_c5mv_details.txt 2>/dev/null
ls -la gpurun_out | head -30
