# fused first panel (small problems): parity + C1/C2 A/B against HEAD
O=gpurun_out/r02fp
mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_lookahead.py tests/test_gpu_golden.py tests/test_gpu_configs.py tests/test_gpu_capi_direct.py -x -q -p no:cacheprovider > $O/pytest.txt 2>&1; echo "pytest rc=$?" >> $O/pytest.txt
for i in 1 2; do
  for v in head new; do
    if [ $v = head ]; then export BGP_LIB_PATH=$PWD/build/ab/libbgp_head.so; else unset BGP_LIB_PATH; fi
    for t in 128 256; do timeout 600 python tools/bench_configs.py --configs 1 --tile $t 2>/dev/null | sed "s/^{/{\"build\": \"$v\", /" >> $O/c1.jsonl; done
  done
done
unset BGP_LIB_PATH
BGP_LIB_PATH=$PWD/build/checked/libbgp.so timeout 900 python tools/sanitize_small.py > $O/checked_sanitize_small.txt 2>&1; echo "checked rc=$?" >> $O/checked_sanitize_small.txt
