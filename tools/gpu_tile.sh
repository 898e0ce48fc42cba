#!/bin/bash
# C4 bench at tile 256 and 512
mkdir -p gpurun_out/tile
for t in ${TILES:-512 256}; do
  timeout 900 python bench.py --tile $t --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/tile/bench_$t.json 2> gpurun_out/tile/bench_$t.err
done
