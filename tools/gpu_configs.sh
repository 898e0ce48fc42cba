#!/bin/bash
O=${CFG_OUT:-gpurun_out/cfg}; mkdir -p $O
for t in ${TILES:-256 512}; do
  timeout 1200 python tools/bench_configs.py --tile $t > $O/configs_$t.jsonl 2> $O/configs_$t.err
done
