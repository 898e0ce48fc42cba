# round 2, second pass: new covariance fast path (parity + bench + ncu),
# the one-process sweep-step tests, sanitizers, and the full CPU evaluation
set -x
O=gpurun_out/r02b
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_golden.py tests/test_gpu_multi.py tests/test_gpu_gp.py -x -q -p no:cacheprovider > $O/pytest.txt 2>&1; echo "pytest rc=$?" >> $O/pytest.txt
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 2 > $O/bench.json 2> $O/bench.err; echo "rc=$?" >> $O/bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
    python bench.py --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline > $O/ncu_bench.log 2>&1; echo "ncu launches rc=$?" >> $O/rc.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:cov_tri -c 1 \
    -o $O/cov_full -f python tools/profile_c4.py --evals 0 > $O/ncu_cov.log 2>&1; echo "ncu cov rc=$?" >> $O/rc.txt
timeout 900 compute-sanitizer --tool memcheck --print-limit 50 python tools/sanitize_small.py > $O/memcheck.txt 2>&1; echo "memcheck rc=$?" >> $O/rc.txt
timeout 900 compute-sanitizer --tool synccheck --print-limit 50 python tools/sanitize_small.py > $O/synccheck.txt 2>&1; echo "synccheck rc=$?" >> $O/rc.txt
timeout 1200 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 50 python tools/sanitize_small.py > $O/racecheck.txt 2>&1; echo "racecheck rc=$?" >> $O/rc.txt
timeout 1500 python tools/cpu_full_eval.py > $O/cpu_full_eval.json 2> $O/cpu_full_eval.err; echo "cpu full rc=$?" >> $O/rc.txt
