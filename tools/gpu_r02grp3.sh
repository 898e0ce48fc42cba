O=${1:-gpurun_out/r02grp3}
mkdir -p $O
BGP_GROUP_DEPTH=6 BGP_PAIR_STEPS=2 timeout 1500 python -m pytest tests/test_gpu_lookahead.py tests/test_gpu_golden.py -x -q -p no:cacheprovider > $O/pytest_d6.txt 2>&1; echo "pytest rc=$?" >> $O/pytest_d6.txt
BGP_GROUP_DEPTH=5 BGP_PAIR_STEPS=2 timeout 600 python tools/stress_sizes.py 1 > $O/stress_d5.txt 2>&1
for i in 1 2; do
  for v in d5:64 d6:64 d5:48 d5:80 d4:48; do
    unset BGP_LIB_PATH BGP_GROUP_DEPTH BGP_PAIR_STEPS
    d=${v%%:*}; k=${v#*:}
    export BGP_GROUP_DEPTH=${d#d} BGP_PAIR_STEPS=$k
    timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 2>/dev/null | tail -1 | sed "s/^{/{\"v\": \"$v\", /" >> $O/c4.jsonl
  done
done
