#!/bin/bash
# GPU-side: one `ncu --set full` capture of one kernel of the bench (tag, kernel regex, extra bench args)
tag=$1; k=$2; shift 2
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 \
    -o gpurun_out/full_${k}_$tag python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e "$@" > gpurun_out/ncu_$tag.log 2>&1
echo "ncu rc=$?"
ncu -i gpurun_out/full_${k}_$tag.ncu-rep --page raw --csv > gpurun_out/raw_${k}_$tag.csv 2>/dev/null
ncu -i gpurun_out/full_${k}_$tag.ncu-rep --page source --csv > gpurun_out/source_${k}_$tag.csv 2>/dev/null
python tools/ncu_summary.py gpurun_out/raw_${k}_$tag.csv
