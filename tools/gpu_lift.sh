#!/bin/bash
mkdir -p gpurun_out
python tools/lift_timing.py > gpurun_out/lift.log 2>&1
KS_KRON_RANK=0 python tools/lift_timing.py >> gpurun_out/lift.log 2>&1
KS_KRON_RANK=0 KS_KRON_MERGE=0 python tools/lift_timing.py >> gpurun_out/lift.log 2>&1
