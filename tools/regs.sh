#!/bin/bash
# registers / stack per kernel instantiation of one .cu (sm_100a): tools/regs.sh csrc/file.cu [filter]
f=$1; k=${2:-kernel}
nvcc --threads 4 -std=c++20 -O3 -lineinfo -Xcompiler -fPIC -I include -I paper_2012_05695_b200/csrc \
  -gencode arch=compute_100a,code=sm_100a -c "$f" -o /tmp/regs_$$.o || exit 1
cuobjdump -res-usage /tmp/regs_$$.o 2>&1 | grep -A1 "Function" | paste - - - | grep "$k" | \
  sed -E 's/.*Function _Z[^ ]*?([a-z0-9_]+_kernel)I([^ ]*)E[^ ]*:.*REG:([0-9]+) STACK:([0-9]+) SHARED:([0-9]+).*/\1 \2 REG=\3 STACK=\4/' | cut -c1-160
rm -f /tmp/regs_$$.o
