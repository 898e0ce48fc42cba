# multi-step tail launch: parity, stress, A/B against one launch per step, C4 regression check
set -x
O=gpurun_out/r02ms
mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_lookahead.py tests/test_gpu_golden.py tests/test_gpu_configs.py tests/test_gpu_capi_direct.py tests/test_gpu_distla.py tests/test_gpu_gp.py -x -q -p no:cacheprovider > $O/pytest.txt 2>&1; echo "pytest rc=$?" >> $O/pytest.txt
for rep in 1 2; do for t in 128 256 512; do timeout 300 python tools/debug_la.py $t 300,700,1000,1500,2523,3000,4100,5000 >> $O/stress.txt 2>&1; done; done
for i in 1 2; do
  for m in 1 0; do
    for t in 128 256; do BGP_MULTI_STEP=$m timeout 600 python tools/bench_configs.py --configs 1,2 --tile $t 2>/dev/null | sed "s/^{/{\"multi\": $m, /" >> $O/ab.jsonl; done
  done
done
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 2 > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/rc.txt
BGP_LIB_PATH=$PWD/build/checked/libbgp.so timeout 900 python tools/sanitize_small.py > $O/checked_sanitize_small.txt 2>&1; echo "checked rc=$?" >> $O/checked_sanitize_small.txt
