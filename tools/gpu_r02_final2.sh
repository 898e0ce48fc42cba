# round 2 final measurement pass on the final code (summaries -> profiles/r02final_*)
set -x
O=${1:-gpurun_out/r02final}
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/nvsmi.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "smoke rc=$?" >> $O/smoke.txt
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/rc.txt
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_reference.json 2> $O/bench_reference.err; echo "ref rc=$?" >> $O/rc.txt
timeout 300 python bench.py --gpus 2 > $O/bench_gpus2_on_1gpu.txt 2>&1; echo "gpus2 rc=$?" >> $O/rc.txt
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
    python bench.py --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline > $O/ncu_bench.log 2>&1; echo "ncu launches rc=$?" >> $O/rc.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_dmma --launch-skip 21 -c 1 \
    -o $O/gemm_full -f python tools/profile_c4.py --evals 0 > $O/ncu_gemm.log 2>&1; echo "ncu gemm rc=$?" >> $O/rc.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:cov_tri -c 1 \
    -o $O/cov_full -f python tools/profile_c4.py --evals 0 > $O/ncu_cov.log 2>&1; echo "ncu cov rc=$?" >> $O/rc.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:trsv_fwd -c 1 \
    -o $O/trsv_full -f python tools/profile_c4.py --evals 0 > $O/ncu_trsv.log 2>&1; echo "ncu trsv rc=$?" >> $O/rc.txt
for t in 128 256 512; do timeout 900 python tools/bench_configs.py --configs 1,2,3,5 --tile $t > $O/configs_tile$t.jsonl 2> $O/configs_tile$t.err; done
timeout 900 python bench.py --workload c5 --steps 1 --warmup 1 > $O/bench_c5_1gpu.json 2> $O/bench_c5.err; echo "c5 rc=$?" >> $O/rc.txt
timeout 900 bash tools/run_reference_tests.sh run $O/reftests.txt > $O/reftests.log 2>&1; echo "reftests rc=$?" >> $O/rc.txt
BGP_LIB_PATH=$PWD/build/checked/libbgp.so timeout 900 python tools/sanitize_small.py > $O/checked_sanitize_small.txt 2>&1; echo "checked rc=$?" >> $O/checked_sanitize_small.txt
