mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${1:-c3}.csv python bench.py --config ${1:-c3} --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/c3l.log 2>&1
echo rc=$?
python tools/launch_agg.py gpurun_out/launches_${1:-c3}.csv
