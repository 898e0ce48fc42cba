#!/bin/bash
# One GPU session: gpu tests, smoke, bench, launch list, ncu --set full of the
# top kernels.  Usage (from the repo root on the box): bash tools/gpu_round.sh TAG
TAG=${1:-r01}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/nvsmi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/rc.txt
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/rc.txt
if [ "${SKIP_NCU:-0}" = "0" ]; then
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
    python bench.py --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline > $O/ncu_bench.log 2>&1; echo "ncu launches rc=$?" >> $O/rc.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_dmma --launch-skip 40 -c 1 \
    -o $O/gemm_full -f python tools/profile_c4.py --evals 0 > $O/ncu_gemm.log 2>&1; echo "ncu gemm rc=$?" >> $O/rc.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:cov_ -c 1 \
    -o $O/cov_full -f python tools/profile_c4.py --evals 0 > $O/ncu_cov.log 2>&1; echo "ncu cov rc=$?" >> $O/rc.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:trsv -c 2 \
    -o $O/trsv_full -f python tools/profile_c4.py --evals 0 > $O/ncu_trsv.log 2>&1; echo "ncu trsv rc=$?" >> $O/rc.txt
fi
