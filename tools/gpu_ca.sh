#!/bin/bash
mkdir -p gpurun_out
timeout 900 python tools/fd_sweep.py 'KS_FD_NAT=0' "KS_LIB_PATH=$PWD/paper_2311_18461_b200/build_ca/libks.so" > gpurun_out/ca_sweep.log 2>&1
KS_LIB_PATH=$PWD/paper_2311_18461_b200/build_ca/libks.so timeout 600 ncu --metrics gpu__time_duration.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum,dram__bytes_read.sum --clock-control none -k regex:"fold" -c 6 --csv \
    --log-file gpurun_out/ca_launches.csv python tools/prof_c3.py c3 > gpurun_out/ca_ncu.log 2>&1
