#!/bin/bash
# GPU-side round check: parity tests, one bench line (with the CPU baseline), the ncu launch
# list of the bench command, and one `ncu --set full` capture per hot kernel.
#   gpurun --timeout 2400 -- bash tools/gpu_round.sh [tag]
tag=${1:-r01}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu_$tag.txt 2>&1
nproc >> gpurun_out/gpu_$tag.txt
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_$tag.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu_$tag.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err
echo "bench rc=$?"; cat gpurun_out/bench_$tag.json; tail -3 gpurun_out/bench_$tag.err
timeout 600 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/bench_ref_$tag.json 2>&1
echo "ref rc=$?"; tail -2 gpurun_out/bench_ref_$tag.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_$tag.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline \
    --no-e2e > gpurun_out/ncu_launch_bench_$tag.log 2>&1
echo "launches rc=$?"
for k in temporal_warp_kernel rows2_kernel cols2_kernel; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 \
      -o gpurun_out/full_${k}_$tag python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e \
      > /dev/null 2>&1
  echo "ncu $k rc=$?"
  ncu -i gpurun_out/full_${k}_$tag.ncu-rep --page raw --csv > gpurun_out/raw_${k}_$tag.csv 2>/dev/null
  ncu -i gpurun_out/full_${k}_$tag.ncu-rep --page details --csv > gpurun_out/details_${k}_$tag.csv 2>/dev/null
  ncu -i gpurun_out/full_${k}_$tag.ncu-rep --page source --csv > gpurun_out/source_${k}_$tag.csv 2>/dev/null
done
ls -la gpurun_out | tail -30
