O=gpurun_out/r02mem
mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_multi.py -x -q -p no:cacheprovider > $O/pytest_multi.txt 2>&1; echo "pytest rc=$?" >> $O/pytest_multi.txt
timeout 900 bash tools/run_reference_tests.sh run $O/reftests.txt > $O/reftests.log 2>&1; echo "reftests rc=$?" >> $O/reftests.log
