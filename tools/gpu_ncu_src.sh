#!/bin/bash
# Full ncu captures of single launches (fused axis-1 stage, matvec pass pair) at
# c3 with the source page (per-line stall samples) exported as CSV.
mkdir -p gpurun_out
python tools/prof_c3.py c3 > gpurun_out/prof_plain.log 2>&1 || exit 1
for spec in "axis1:k_fd_axis1:1:1" "mvA:ks_pair:26:1" "mvB:ks_pair:27:1" "xf:k_xfold:5:1"; do
  IFS=: read name rx skip cnt <<< "$spec"
  timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:"$rx" -s $skip -c $cnt \
      -o /tmp/prof_$name python tools/prof_c3.py c3 > gpurun_out/ncu_$name.log 2>&1
  python tools/ncu_summary.py /tmp/prof_$name.ncu-rep gpurun_out/ncu_${name}_summary.csv >> gpurun_out/ncu_$name.log 2>&1
  ncu -i /tmp/prof_$name.ncu-rep --page raw --csv > gpurun_out/ncu_${name}_raw.csv 2>/dev/null
  ncu -i /tmp/prof_$name.ncu-rep --page source --csv > gpurun_out/ncu_${name}_source.csv 2>/dev/null
  ncu -i /tmp/prof_$name.ncu-rep --page details > gpurun_out/ncu_${name}_details.txt 2>/dev/null
done
ls -la gpurun_out
