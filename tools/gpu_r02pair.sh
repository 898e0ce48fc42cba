# step pairs (k = 2b merged update): parity with pairs forced on small sizes, C4 A/B
O=${1:-gpurun_out/r02pair}
mkdir -p $O
BGP_PAIR_STEPS=4 timeout 1500 python -m pytest tests/test_gpu_lookahead.py tests/test_gpu_golden.py tests/test_gpu_configs.py -x -q -p no:cacheprovider > $O/pytest_pairs_forced.txt 2>&1; echo "pytest rc=$?" >> $O/pytest_pairs_forced.txt
BGP_PAIR_STEPS=4 timeout 600 python tools/stress_sizes.py 1 > $O/stress_pairs_forced.txt 2>&1
BGP_PAIR_STEPS=4 BGP_LIB_PATH=$PWD/build/checked/libbgp.so timeout 900 python tools/sanitize_small.py > $O/checked_sanitize_small.txt 2>&1; echo "checked rc=$?" >> $O/checked_sanitize_small.txt
for i in 1 2; do
  for v in head new64 new80 new100; do
    unset BGP_LIB_PATH BGP_PAIR_STEPS
    if [ $v = head ]; then export BGP_LIB_PATH=$PWD/build/ab/libbgp_head.so; fi
    if [ $v != head ]; then export BGP_PAIR_STEPS=${v#new}; fi
    timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 2>/dev/null | tail -1 | sed "s/^{/{\"v\": \"$v\", /" >> $O/c4.jsonl
  done
done
