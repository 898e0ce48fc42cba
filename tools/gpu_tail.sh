#!/bin/bash
# sweep the re-tiled tail size on the C4 bench: TILE=512 TAILS="..." bash tools/gpu_tail.sh
O=gpurun_out/tail; mkdir -p $O
TILE=${TILE:-512}
for t in ${TAILS:-0 8 16 24 32 48}; do
  BGP_TAIL=$t timeout 600 python bench.py --tile $TILE --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 \
    > $O/b${TILE}_$t.json 2> $O/b${TILE}_$t.err
done
