O=${1:-gpurun_out/r02grp2}
mkdir -p $O
BGP_GROUP_DEPTH=4 BGP_PAIR_STEPS=2 timeout 1500 python -m pytest tests/test_gpu_lookahead.py tests/test_gpu_golden.py tests/test_gpu_configs.py -x -q -p no:cacheprovider > $O/pytest_d4.txt 2>&1; echo "pytest rc=$?" >> $O/pytest_d4.txt
BGP_GROUP_DEPTH=4 BGP_PAIR_STEPS=2 BGP_LIB_PATH=$PWD/build/checked/libbgp.so timeout 900 python tools/sanitize_small.py > $O/checked_sanitize_small.txt 2>&1; echo "checked rc=$?" >> $O/checked_sanitize_small.txt
for i in 1 2 3; do
  for v in head d2 d4 d5; do
    unset BGP_LIB_PATH BGP_GROUP_DEPTH
    if [ $v = head ]; then export BGP_LIB_PATH=$PWD/build/ab/libbgp_head.so; else export BGP_GROUP_DEPTH=${v#d}; fi
    timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 2>/dev/null | tail -1 | sed "s/^{/{\"v\": \"$v\", /" >> $O/c4.jsonl
  done
done
