#!/bin/bash
# sweep the re-tiled tail size on the C4 bench
mkdir -p gpurun_out/tail
for t in ${TAILS:-0 8 16 24 32 48}; do
  BGP_TAIL=$t timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/tail/b_$t.json 2> gpurun_out/tail/b_$t.err
done
