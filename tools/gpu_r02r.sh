# substitution panel solve in chain-bound steps: correctness + C1/C2/C4
set -x
O=gpurun_out/r02r
mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_lookahead.py tests/test_gpu_golden.py tests/test_gpu_configs.py tests/test_gpu_capi_direct.py tests/test_gpu_gp.py tests/test_gpu_distla.py -x -q -p no:cacheprovider > $O/pytest.txt 2>&1; echo "pytest rc=$?" >> $O/pytest.txt
BGP_LIB_PATH=$PWD/build/checked/libbgp.so timeout 900 python tools/sanitize_small.py > $O/checked_sanitize_small.txt 2>&1; echo "checked rc=$?" >> $O/rc.txt
for t in 256 512; do timeout 600 python tools/bench_configs.py --configs 1,2 --tile $t > $O/c12_tile$t.jsonl 2> $O/c12_tile$t.err; done
BGP_TRSM_SUBST=0 timeout 600 python tools/bench_configs.py --configs 1,2 --tile 256 > $O/c12_tile256_nosubst.jsonl 2> $O/c12_nosubst.err
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $O/bench.json 2> $O/bench.err
