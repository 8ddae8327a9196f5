#!/bin/bash
# Round-end style measurement pass: GPU tests, smoke, bench (c3 default, c5),
# reference arm, c4 sweep, ncu launch list of the bench command, ncu --set full
# capture of the FD / matvec kernels (summarised to CSV on the box: the
# reports themselves exceed gpurun's 64 MiB return limit). SKIP_TESTS=1 skips pytest, ONLY_NCU=1 runs only the full captures.
mkdir -p gpurun_out
if [ -z "$ONLY_NCU" ]; then
if [ -z "$SKIP_TESTS" ]; then
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_gpu.log
fi
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench.log 2>&1
echo "rc=$?" >> gpurun_out/bench.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1
timeout 900 python bench.py --config c5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c5.log 2>&1
timeout 900 python tools/c4_sweep.py > gpurun_out/c4_sweep.jsonl 2> gpurun_out/c4_sweep.err
python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-solve > gpurun_out/bench_small.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-solve > gpurun_out/ncu_launch.log 2>&1
fi
python tools/prof_c3.py c3 > gpurun_out/prof_plain.log 2>&1
for spec in "fd:k_xfold|k_fd_axis1:5:5" "mv:ks_pair:26:2"; do
  IFS=: read name rx skip cnt <<< "$spec"
  timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:"$rx" -s $skip -c $cnt \
      -o /tmp/prof_$name python tools/prof_c3.py c3 > gpurun_out/ncu_$name.log 2>&1
  python tools/ncu_summary.py /tmp/prof_$name.ncu-rep gpurun_out/ncu_${name}_summary.csv >> gpurun_out/ncu_$name.log 2>&1
  ncu -i /tmp/prof_$name.ncu-rep --page raw --csv > gpurun_out/ncu_${name}_raw.csv 2>/dev/null
done
echo "done" >> gpurun_out/ncu_mv.log
