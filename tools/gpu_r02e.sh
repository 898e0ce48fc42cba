# round 2, fifth pass: pipelined theta sweep (C2), gathered dist tail, cov u8
set -x
O=gpurun_out/r02e
mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_gp.py tests/test_gpu_multi.py tests/test_gpu_golden.py -x -q -p no:cacheprovider > $O/pytest.txt 2>&1; echo "pytest rc=$?" >> $O/pytest.txt
for t in 256 128; do timeout 600 python tools/bench_configs.py --configs 2 --tile $t > $O/c2_tile$t.jsonl 2> $O/c2_tile$t.err; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:cov_tri \
     python tools/profile_c4.py --evals 1 > $O/cov_u8.csv 2> $O/cov_u8.err
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 2 > $O/bench.json 2> $O/bench.err; echo "rc=$?" >> $O/bench.err
