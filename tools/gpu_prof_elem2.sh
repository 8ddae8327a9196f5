python tools/prof_c3.py c3 > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_kron_elem" -s 1 -c 1 -o gpurun_out/prof_elem2 python tools/prof_c3.py c3 > gpurun_out/ncu_elem2.log 2>&1
