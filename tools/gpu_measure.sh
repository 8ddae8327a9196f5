#!/bin/bash
# Round-end style measurement pass: GPU tests, smoke, bench (c3 default incl. legs),
# reference arm, c4 sweep, ncu launch list of the bench command, ncu --set full
# captures of the FD kernels (k_xfold, k_fd_axis1) and of the matvec pass pairs
# (ks_pairt, ks_pairb), summarised to CSV on the box (the reports exceed gpurun's
# 64 MiB return limit). SKIP_TESTS=1 skips pytest, ONLY_NCU=1 runs only the captures.
mkdir -p gpurun_out
if [ -z "$ONLY_NCU" ]; then
if [ -z "$SKIP_TESTS" ]; then
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_gpu.log
fi
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1
echo "rc=$?" >> gpurun_out/bench.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1
timeout 900 python tools/c4_sweep.py > gpurun_out/c4_sweep.jsonl 2> gpurun_out/c4_sweep.err
python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-solve --no-extra > gpurun_out/bench_small.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 600 --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-solve --no-extra > gpurun_out/ncu_launch.log 2>&1
fi
python tools/prof_c3.py c3 > gpurun_out/prof_plain.log 2>&1
# the matvec pair kernels of the last apply: count the launches first (the first apply times the candidates)
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"ks_pair" --csv \
    --log-file gpurun_out/mv_launches.csv python tools/prof_c3.py c3 > /dev/null 2>&1
nmv=$(grep -c "ks_pair" gpurun_out/mv_launches.csv)
mvskip=$((nmv - 2))
for spec in "fd:k_xfold|k_fd_axis1:5:5" "mv:ks_pair:$mvskip:2"; do
  IFS=: read name rx skip cnt <<< "$spec"
  timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:"$rx" -s $skip -c $cnt \
      -o /tmp/prof_$name python tools/prof_c3.py c3 > gpurun_out/ncu_$name.log 2>&1
  python tools/ncu_summary.py /tmp/prof_$name.ncu-rep gpurun_out/ncu_${name}_summary.csv >> gpurun_out/ncu_$name.log 2>&1
done
bash tools/gpu_c5ncu2.sh
bash tools/gpu_c5prof.sh
echo "done" >> gpurun_out/ncu_mv.log
