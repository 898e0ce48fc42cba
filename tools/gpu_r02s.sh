set -x
O=gpurun_out/r02s
mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_multi.py tests/test_gpu_lookahead.py tests/test_gpu_configs.py -x -q -p no:cacheprovider > $O/pytest.txt 2>&1; echo "pytest rc=$?" >> $O/pytest.txt
BGP_LIB_PATH=$PWD/build/checked/libbgp.so timeout 900 python tools/sanitize_small.py > $O/checked_sanitize_small.txt 2>&1; echo "checked rc=$?" >> $O/rc.txt
BGP_LIB_PATH=$PWD/build/checked/libbgp.so timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -p no:cacheprovider -k "one_process or gathered_tail" > $O/checked_multi.txt 2>&1; echo "checked multi rc=$?" >> $O/rc.txt
