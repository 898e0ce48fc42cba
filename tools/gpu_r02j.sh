# CPU baseline: sub-evaluation sampler vs a second timed full evaluation
set -x
O=gpurun_out/r02j
mkdir -p $O
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/rc.txt
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_reference.json 2> $O/bench_reference.err; echo "ref rc=$?" >> $O/rc.txt
timeout 1500 python tools/cpu_full_eval.py > $O/cpu_full_eval.json 2> $O/cpu_full_eval.err; echo "cpu full rc=$?" >> $O/rc.txt
