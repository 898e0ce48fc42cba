# L2-ordered trailing update: parity, C4 bench, one update launch under ncu
set -x
O=gpurun_out/r02l2
mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_lookahead.py tests/test_gpu_golden.py tests/test_gpu_configs.py -x -q -p no:cacheprovider > $O/pytest.txt 2>&1; echo "pytest rc=$?" >> $O/pytest.txt
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 2 > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/rc.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_dmma --launch-skip 21 -c 1 \
    -o $O/gemm_full -f python tools/profile_c4.py --evals 0 > $O/ncu_gemm.log 2>&1; echo "ncu gemm rc=$?" >> $O/rc.txt
timeout 600 python tools/bench_configs.py --configs 2,3 --tile 256 > $O/configs_tile256.jsonl 2> $O/configs.err
