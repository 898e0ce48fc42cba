#!/bin/bash
mkdir -p gpurun_out/cfg
for t in ${TILES:-256 512}; do
  timeout 1200 python tools/bench_configs.py --tile $t > gpurun_out/cfg/configs_$t.jsonl 2> gpurun_out/cfg/configs_$t.err
done
