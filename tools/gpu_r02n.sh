# covariance fast path on padded tiles too: parity + ncu duration
set -x
O=gpurun_out/r02n
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_golden.py tests/test_gpu_configs.py tests/test_gpu_gp.py tests/test_gpu_distla.py -x -q -p no:cacheprovider > $O/pytest.txt 2>&1; echo "pytest rc=$?" >> $O/pytest.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:cov_tri \
     python tools/profile_c4.py --evals 2 > $O/cov.csv 2> $O/cov.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:cov_tri -c 1 \
    -o $O/cov_full -f python tools/profile_c4.py --evals 0 > $O/ncu_cov.log 2>&1; echo "ncu cov rc=$?" >> $O/rc.txt
BGP_LIB_PATH=$PWD/build/checked/libbgp.so timeout 900 python tools/sanitize_small.py > $O/checked_sanitize_small.txt 2>&1; echo "checked rc=$?" >> $O/rc.txt
