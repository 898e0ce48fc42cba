#!/bin/bash
# look-ahead robustness: many small/ragged factorizations at every tile size
mkdir -p gpurun_out/stress
for rep in 1 2 3; do
  for t in 128 256 512; do
    timeout 300 python tools/debug_la.py $t 300,700,1000,1500,2523,3000,4100,5000 >> gpurun_out/stress/log.txt 2>&1
  done
done
grep -c relerr gpurun_out/stress/log.txt > gpurun_out/stress/count.txt
grep -v relerr gpurun_out/stress/log.txt | head -20 >> gpurun_out/stress/count.txt
