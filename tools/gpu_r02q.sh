set -x
O=gpurun_out/r02q
mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_multi.py -x -q -p no:cacheprovider > $O/pytest.txt 2>&1; echo "pytest rc=$?" >> $O/pytest.txt
