#!/bin/bash
# GPU-side: sharded arm at world size 1 (C2, C4), the release gate x10 (criterion 5 robustness)
mkdir -p gpurun_out
for cfg in c2 c4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 \
      --master-port 29511 bench.py --gpus 1 --sharded --config $cfg --steps 5 --warmup 3 \
      > gpurun_out/sharded_${cfg}_world1.json 2> gpurun_out/sharded_${cfg}.err
  echo "sharded $cfg rc=$?"; tail -c 600 gpurun_out/sharded_${cfg}_world1.json; echo
done
pass=0
for i in $(seq 1 10); do
  timeout 300 ./oracle/_ref/release_gate > gpurun_out/gate_run_$i.log 2>&1 && pass=$((pass+1))
  grep -E "FAIL" gpurun_out/gate_run_$i.log
done
echo "release gate 9/9 in $pass of 10 runs"
