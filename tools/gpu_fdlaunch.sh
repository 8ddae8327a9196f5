#!/bin/bash
# per-kernel FD launch list (c3, 3 applications) + full capture of the transforms of one application
mkdir -p gpurun_out
python tools/prof_c3.py c3 > gpurun_out/fdl_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_write.sum --clock-control none --csv \
    -k regex:"k_mode_gemm_fold|k_fd_solve" --log-file gpurun_out/fd_launches.csv python tools/prof_c3.py c3 > gpurun_out/fdl_ncu.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_mode_gemm_fold" -s 6 -c 6 \
    -o gpurun_out/prof_fd python tools/prof_c3.py c3 > gpurun_out/fdl_full.log 2>&1
echo done >> gpurun_out/fdl_full.log
