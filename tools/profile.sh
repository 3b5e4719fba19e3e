#!/bin/bash
# usage: tools_profile.sh <kernel-regex> <tag> [skip]  -- ncu full capture of one launch of the bench
k=$1; tag=$2; skip=${3:-1}
ncu --set full --clock-control none --import-source on -k regex:$k -s $skip -c 1 -o gpurun_out/p_$tag python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
ncu -i gpurun_out/p_$tag.ncu-rep --page raw --csv > gpurun_out/raw_$tag.csv
ncu -i gpurun_out/p_$tag.ncu-rep --page details --csv > gpurun_out/details_$tag.csv
ncu -i gpurun_out/p_$tag.ncu-rep --page source --csv --print-source cuda > gpurun_out/srccuda_$tag.csv 2>/dev/null; ncu -i gpurun_out/p_$tag.ncu-rep --page source --csv > gpurun_out/source_$tag.csv 2>/dev/null
rm -f gpurun_out/p_$tag.ncu-rep
