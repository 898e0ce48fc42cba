#!/bin/bash
# Quick GPU check: gpu tests, kernel micro-timings, short bench (no ncu).
# Usage: bash tools/gpu_quick.sh TAG [pytest -k expr]
TAG=${1:-q}
O=gpurun_out/$TAG
mkdir -p $O
if [ -n "$2" ]; then K="-k $2"; else K=""; fi
timeout 600 python -m pytest tests -m gpu -x -q $K > $O/pytest.log 2>&1; echo "pytest rc=$?" > $O/rc.txt
timeout 300 python tools/kbench.py > $O/kbench.log 2>&1; echo "kbench rc=$?" >> $O/rc.txt
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/rc.txt
