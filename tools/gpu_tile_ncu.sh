#!/bin/bash
# full captures (source page) of the tile kernel at c5 (kept by timing) and c3 (forced)
mkdir -p gpurun_out
for cfg in c5 c3; do
  if [ $cfg = c5 ]; then cmd="python tools/prof_c5mv.py"; export KS_KRON_JIT=log; export KS_KRON_TILE="22,3,2,8,2,3"; else export KS_KRON_TILE="22,3,2,8,2,1"; cmd="python tools/prof_c3.py c3"; export KS_KRON_JIT=tile; fi
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"ks_pair" --csv \
      --log-file gpurun_out/${cfg}t_launches.csv $cmd > /dev/null 2>&1
  n=$(grep -c "ks_pairt" gpurun_out/${cfg}t_launches.csv)
  timeout 1200 ncu -f --set full --clock-control none --import-source on -k regex:"ks_pairt" -s $((n - 1)) -c 1 \
      -o /tmp/prof_${cfg}t $cmd > gpurun_out/ncu_${cfg}t.log 2>&1
  python tools/ncu_summary.py /tmp/prof_${cfg}t.ncu-rep gpurun_out/ncu_${cfg}t_summary.csv >> gpurun_out/ncu_${cfg}t.log 2>&1
  ncu -i /tmp/prof_${cfg}t.ncu-rep --page source --csv > gpurun_out/ncu_${cfg}t_source.csv 2>/dev/null
  ncu -i /tmp/prof_${cfg}t.ncu-rep --page details > gpurun_out/ncu_${cfg}t_details.txt 2>/dev/null
done
ls -la gpurun_out | head -40
