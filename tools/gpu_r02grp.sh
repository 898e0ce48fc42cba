# step groups of depth d (d panels merged in the group's last launch): parity with groups forced, C4 A/B
O=${1:-gpurun_out/r02grp}
mkdir -p $O
for d in 3 4; do
  BGP_GROUP_DEPTH=$d BGP_PAIR_STEPS=2 timeout 1500 python -m pytest tests/test_gpu_lookahead.py tests/test_gpu_golden.py -x -q -p no:cacheprovider > $O/pytest_d$d.txt 2>&1; echo "pytest rc=$?" >> $O/pytest_d$d.txt
  BGP_GROUP_DEPTH=$d BGP_PAIR_STEPS=2 timeout 600 python tools/stress_sizes.py 1 > $O/stress_d$d.txt 2>&1
  BGP_GROUP_DEPTH=$d timeout 900 python tools/residual_sizes.py 40000,67275 512 > $O/residual_d$d.jsonl 2>&1
done
BGP_GROUP_DEPTH=3 BGP_PAIR_STEPS=2 BGP_LIB_PATH=$PWD/build/checked/libbgp.so timeout 900 python tools/sanitize_small.py > $O/checked_sanitize_small.txt 2>&1; echo "checked rc=$?" >> $O/checked_sanitize_small.txt
for i in 1 2; do
  for v in head d2 d3 d4; do
    unset BGP_LIB_PATH BGP_GROUP_DEPTH
    if [ $v = head ]; then export BGP_LIB_PATH=$PWD/build/ab/libbgp_head.so; else export BGP_GROUP_DEPTH=${v#d}; fi
    timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 2>/dev/null | tail -1 | sed "s/^{/{\"v\": \"$v\", /" >> $O/c4.jsonl
  done
done
