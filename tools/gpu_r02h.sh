# padding skip in the sweep's last tile row; regression + bench
set -x
O=gpurun_out/r02h
mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_lookahead.py tests/test_gpu_golden.py tests/test_gpu_configs.py tests/test_gpu_capi_direct.py tests/test_gpu_distla.py -x -q -p no:cacheprovider > $O/pytest.txt 2>&1; echo "pytest rc=$?" >> $O/pytest.txt
BGP_LIB_PATH=$PWD/build/checked/libbgp.so timeout 900 python tools/sanitize_small.py > $O/checked_sanitize_small.txt 2>&1; echo "checked rc=$?" >> $O/rc.txt
for i in 1 2; do timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 2 > $O/bench$i.json 2> $O/bench$i.err; done
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 --tile 256 > $O/bench_t256.json 2> $O/bench_t256.err
