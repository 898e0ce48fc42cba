#!/bin/bash
# GPU tests, then compare Cholesky variants on the C4 bench:
#   BGP_LOOKAHEAD=0/1/2 (sequential / look-ahead / sequential on 147 SMs), BGP_TRSM=0/1
mkdir -p gpurun_out/la
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/la/pytest.log 2>&1; echo "pytest rc=$?" > gpurun_out/la/rc.txt
for cfg in ${CFGS:-"1 1" "1 0"}; do
  set -- $cfg
  BGP_LOOKAHEAD=$1 BGP_TRSM=$2 timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 \
    > gpurun_out/la/bench_$1$2.json 2> gpurun_out/la/bench_$1$2.err
done
