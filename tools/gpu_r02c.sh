# round 2, third pass: full-size parity suite, covariance fast path v2,
# C2 profile + tail experiments, the reference's own tests via the alias,
# and an ncu capture of the 256 tile POTRF (+ inverse)
set -x
O=gpurun_out/r02c
mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_configs.py tests/test_gpu_golden.py tests/test_gpu_capi_direct.py tests/test_gpu_cli.py -x -q -p no:cacheprovider > $O/pytest.txt 2>&1; echo "pytest rc=$?" >> $O/pytest.txt
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 2 > $O/bench.json 2> $O/bench.err; echo "rc=$?" >> $O/bench.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:cov_tri -c 1 \
    -o $O/cov_full -f python tools/profile_c4.py --evals 0 > $O/ncu_cov.log 2>&1; echo "ncu cov rc=$?" >> $O/rc.txt
for t in 256 128; do timeout 600 python tools/bench_configs.py --configs 2 --tile $t > $O/c2_tile$t.jsonl 2> $O/c2_tile$t.err; done
for tl in 48 64; do BGP_TAIL=$tl timeout 600 python tools/bench_configs.py --configs 2 --tile 256 > $O/c2_tile256_tail$tl.jsonl 2> $O/c2_tail$tl.err; done
timeout 900 bash tools/run_reference_tests.sh run $O/reftests.txt > $O/reftests.log 2>&1; echo "reftests rc=$?" >> $O/rc.txt
timeout 600 python tools/potrf_bench.py > $O/potrf_bench.jsonl 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tile_potrf -c 1 --launch-skip 60 \
    -o $O/potrf256_full -f python tools/potrf_bench.py > $O/ncu_potrf.log 2>&1; echo "ncu potrf rc=$?" >> $O/rc.txt
