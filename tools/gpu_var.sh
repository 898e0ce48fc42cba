#!/bin/bash
# C4 bench with probe variants of the BK=32 GEMM (forced through the bk16 slot)
mkdir -p gpurun_out/var
for v in ${VARIANTS:-BK32 BK32_NOSTAG BK32_EVN}; do
  BGP_GEMM_CFG=16 BGP_LIB_PATH=$PWD/build/probe/libbgp_$v.so timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/var/b_$v.json 2> gpurun_out/var/b_$v.err
done
