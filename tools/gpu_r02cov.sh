# K1 with pre-scaled points, 256-entry exp table: parity + ncu + bench
O=${1:-gpurun_out/r02cov}
mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_golden.py tests/test_gpu_configs.py tests/test_gpu_distla.py tests/test_gpu_gp.py -x -q -p no:cacheprovider > $O/pytest.txt 2>&1; echo "pytest rc=$?" >> $O/pytest.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:cov_tri -c 1 \
    -o $O/cov_full -f python tools/profile_c4.py --evals 0 > $O/ncu_cov.log 2>&1; echo "ncu cov rc=$?" >> $O/rc.txt
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/rc.txt
BGP_LIB_PATH=$PWD/build/checked/libbgp.so timeout 900 python tools/sanitize_small.py > $O/checked_sanitize_small.txt 2>&1; echo "checked rc=$?" >> $O/checked_sanitize_small.txt
