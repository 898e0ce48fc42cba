#!/bin/bash
# Build probe variants of libbgp (experiment macros in gemm.cu) and time them.
# Usage: bash tools/gemm_probe.sh build   (here)   |   bash tools/gemm_probe.sh run (GPU box)
set -e
D=build/probe
if [ "$1" = "build" ]; then
  mkdir -p $D
  for v in ${VARIANTS:-base NO_TMA NO_EPI NO_TMA_NO_EPI NO_BAR}; do
    case $v in
      base) F="";; NO_TMA) F="-DBGP_EXP_NO_TMA";; NO_EPI) F="-DBGP_EXP_NO_EPI";;
      NO_TMA_NO_EPI) F="-DBGP_EXP_NO_TMA -DBGP_EXP_NO_EPI";;
      TRACE) F="-DBGP_EXP_TRACE";;
      BK32) F="-DBGP_GEMM_BK32";;
      BK32_SLICE) F="-DBGP_GEMM_BK32 -DBGP_EXP_EPI_SLICE";;
      BK32_SLICE_TRACE) F="-DBGP_GEMM_BK32 -DBGP_EXP_EPI_SLICE -DBGP_EXP_TRACE";;
      BK16S2) F="-DBGP_GEMM_BK16S2";;
      BK16S2_TRACE) F="-DBGP_GEMM_BK16S2 -DBGP_EXP_TRACE";;
      BK32_RED) F="-DBGP_GEMM_BK32 -DBGP_EPI_RED";;
      BK32_RED_TRACE) F="-DBGP_GEMM_BK32 -DBGP_EPI_RED -DBGP_EXP_TRACE";;
      BK32_CORE) F="-DBGP_GEMM_BK32 -DBGP_EXP_NO_TMA -DBGP_EXP_NO_EPI";;
      BK32_CORE_NW) F="-DBGP_GEMM_BK32 -DBGP_EXP_NO_TMA -DBGP_EXP_NO_EPI -DBGP_EXP_NO_STAGE_WAIT";;
      BK16_CORE) F="-DBGP_EXP_NO_TMA -DBGP_EXP_NO_EPI";;
      BK16_CORE_NW) F="-DBGP_EXP_NO_TMA -DBGP_EXP_NO_EPI -DBGP_EXP_NO_STAGE_WAIT";;
      BK32_STORE) F="-DBGP_GEMM_BK32 -DBGP_EXP_STORE_EPI";;
      BK32_ONE) F="-DBGP_GEMM_BK32 -DBGP_EXP_ONE_GROUP";;
      BK32_ONE_CORE) F="-DBGP_GEMM_BK32 -DBGP_EXP_ONE_GROUP -DBGP_EXP_NO_TMA -DBGP_EXP_NO_EPI";;
      G3) F="-DBGP_GEMM_3G";;
      G3_CORE) F="-DBGP_GEMM_3G -DBGP_EXP_NO_TMA -DBGP_EXP_NO_EPI";;
      BK32_TRACE) F="-DBGP_GEMM_BK32 -DBGP_EXP_TRACE";;
      BK32_STRACE) F="-DBGP_GEMM_BK32 -DBGP_EXP_STRACE";;
      BK32_NOSTAG) F="-DBGP_GEMM_BK32 -DBGP_EXP_NO_STAGGER";;
      BK32_EVN) F="-DBGP_GEMM_BK32 -DBGP_EXP_EVICT_NORMAL";;
      NO_BAR_TRACE) F="-DBGP_EXP_NO_TMA -DBGP_EXP_NO_EPI -DBGP_EXP_NO_BAR -DBGP_EXP_TRACE";;
      NO_BAR) F="-DBGP_EXP_NO_TMA -DBGP_EXP_NO_EPI -DBGP_EXP_NO_BAR";;
    esac
    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC $F $EXTRA \
      -c paper_1305_4886_b200/csrc/gemm.cu -o $D/gemm_$v.o
    nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $D/libbgp_$v.so build/capi.o build/cov.o \
      build/potrf.o $D/gemm_$v.o build/solve.o build/rng.o build/trsv.o build/gemm_bk32.o
  done
else
  mkdir -p gpurun_out/probe
  L=""; for v in ${VARIANTS:-base NO_TMA NO_EPI NO_TMA_NO_EPI NO_BAR}; do L="$L $D/libbgp_$v.so"; done
  python tools/gemm_probe.py $L 2>&1 | tee gpurun_out/probe/gemm_probe.log
fi
