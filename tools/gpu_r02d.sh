# round 2, fourth pass: covariance variants (unroll 4 / 8, underflow test
# dropped from the host's distance bound), checked-build dataflow runs
set -x
O=gpurun_out/r02d
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_golden.py tests/test_gpu_configs.py tests/test_gpu_gp.py -x -q -p no:cacheprovider > $O/pytest.txt 2>&1; echo "pytest rc=$?" >> $O/pytest.txt
for v in prod u8; do
  if [ $v = prod ]; then LIB=$PWD/paper_1305_4886_b200/libbgp.so; else LIB=$PWD/build/var_$v/libbgp.so; fi
  BGP_LIB_PATH=$LIB timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:cov_tri \
     python tools/profile_c4.py --evals 1 > $O/cov_$v.csv 2> $O/cov_$v.err
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:cov_tri -c 1 \
    -o $O/cov_full -f python tools/profile_c4.py --evals 0 > $O/ncu_cov.log 2>&1; echo "ncu cov rc=$?" >> $O/rc.txt
BGP_LIB_PATH=$PWD/build/checked/libbgp.so timeout 900 python tools/sanitize_small.py > $O/checked_sanitize_small.txt 2>&1; echo "checked rc=$?" >> $O/rc.txt
BGP_LIB_PATH=$PWD/build/checked/libbgp.so timeout 900 python -m pytest tests/test_gpu_lookahead.py tests/test_gpu_multi.py tests/test_gpu_capi_direct.py -x -q -p no:cacheprovider > $O/checked_pytest.txt 2>&1; echo "checked pytest rc=$?" >> $O/rc.txt
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 2 > $O/bench.json 2> $O/bench.err; echo "rc=$?" >> $O/bench.err
