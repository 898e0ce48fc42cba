#!/bin/bash
# Round profile set: full bench (with CPU baseline), ncu launch list of the
# bench command, ncu --set full of the trailing-update GEMM, cov build, and
# forward solve.  The look-ahead lives inside each update launch, so the
# schedule under ncu (kernels serialised) is the production one.
TAG=${1:-r01c}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/nvsmi.txt 2>&1
timeout 60 ncu --metrics gpu__time_duration.sum -c 1 env > $O/ncu_env.txt 2>&1
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/rc.txt
# the look-ahead waits are inside one launch, so it stays on under ncu
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
    python bench.py --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline > $O/ncu_bench.log 2>&1; echo "ncu launches rc=$?" >> $O/rc.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_dmma --launch-skip 21 -c 1 \
    -o $O/gemm_full -f python tools/profile_c4.py --evals 0 > $O/ncu_gemm.log 2>&1; echo "ncu gemm rc=$?" >> $O/rc.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:cov_ -c 1 \
    -o $O/cov_full -f python tools/profile_c4.py --evals 0 > $O/ncu_cov.log 2>&1; echo "ncu cov rc=$?" >> $O/rc.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:trsv_fwd -c 1 \
    -o $O/trsv_full -f python tools/profile_c4.py --evals 0 > $O/ncu_trsv.log 2>&1; echo "ncu trsv rc=$?" >> $O/rc.txt
