#!/bin/bash
# GPU round plus the C3 / C4 bench lines and the sharded C4 pass at world size 1:
#   gpurun --timeout 3000 -- bash tools/gpu_round_cfg.sh <tag>
tag=${1:-r02}
bash tools/gpu_round.sh $tag
for cfg in c3 c4; do
  steps=3; [ $cfg = c4 ] && steps=2
  timeout 900 python bench.py --config $cfg --steps $steps --warmup 3 > gpurun_out/${tag}_$cfg.json 2> gpurun_out/${tag}_$cfg.err
  echo "bench $cfg rc=$?"; tail -c 400 gpurun_out/${tag}_$cfg.json; echo
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 \
    --master-port 29511 bench.py --gpus 1 --sharded --config c4 --steps 2 --warmup 3 \
    > gpurun_out/${tag}_sharded_c4.json 2> gpurun_out/${tag}_sharded_c4.err
echo "sharded c4 rc=$?"; tail -c 400 gpurun_out/${tag}_sharded_c4.json
