set -x
O=gpurun_out/r02w2
mkdir -p $O
timeout 120 tools/probes/potrf_trace > $O/potrf_trace.jsonl 2>&1; echo "rc=$?" >> $O/potrf_trace.jsonl
timeout 1500 python -m pytest tests/test_gpu_lookahead.py tests/test_gpu_golden.py tests/test_gpu_capi_direct.py tests/test_gpu_distla.py -x -q -p no:cacheprovider > $O/pytest.txt 2>&1; echo "pytest rc=$?" >> $O/pytest.txt
for t in 128 256; do timeout 600 python tools/bench_configs.py --configs 1,2 --tile $t > $O/c12_tile$t.jsonl 2> $O/c12_tile$t.err; done
BGP_LIB_PATH=$PWD/build/checked/libbgp.so timeout 900 python tools/sanitize_small.py > $O/checked_sanitize_small.txt 2>&1; echo "checked rc=$?" >> $O/checked_sanitize_small.txt
