# round 2, sixth pass: tile POTRF with the diagonal chain overlapping the
# sub-panel solve; C2 sequential / pipelined (2, 3 lanes); the dist tail
set -x
O=gpurun_out/r02f
mkdir -p $O
timeout 600 python tools/potrf_bench.py > $O/potrf_bench.jsonl 2>&1
timeout 1500 python -m pytest tests/test_gpu_lookahead.py tests/test_gpu_multi.py tests/test_gpu_golden.py tests/test_gpu_gp.py tests/test_gpu_configs.py -x -q -p no:cacheprovider > $O/pytest.txt 2>&1; echo "pytest rc=$?" >> $O/pytest.txt
for t in 256 128; do timeout 600 python tools/bench_configs.py --configs 1,2 --tile $t > $O/c12_tile$t.jsonl 2> $O/c12_tile$t.err; done
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 2 > $O/bench.json 2> $O/bench.err; echo "rc=$?" >> $O/bench.err
