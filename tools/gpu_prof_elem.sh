python tools/prof_c3.py c3 > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_kron_elem" -c 4 -o gpurun_out/prof_elem python tools/prof_c3.py c3 > gpurun_out/ncu_elem.log 2>&1
