#!/bin/bash
# ncu --set full of one probe-variant GEMM launch each (see gemm_probe.sh)
D=build/probe
mkdir -p gpurun_out/probe
for v in ${@:-base NO_TMA_NO_EPI}; do
  PROBE_REPS=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_dmma -s 1 -c 1 \
    -o gpurun_out/probe/ncu_$v -f python tools/gemm_probe.py $D/libbgp_$v.so > gpurun_out/probe/ncu_$v.log 2>&1
done
