# A/B against the round-1 tree (build/r01_tree, not committed): C5 and C4 at tile 512
set -x
O=$PWD/gpurun_out/r02k
mkdir -p $O
for i in 1 2; do
  (cd build/r01_tree && timeout 600 python tools/bench_configs.py --configs 5 --tile 512 > $O/c5_r01_$i.jsonl 2> $O/c5_r01_$i.err)
  timeout 600 python tools/bench_configs.py --configs 5 --tile 512 > $O/c5_r02_$i.jsonl 2> $O/c5_r02_$i.err
done
(cd build/r01_tree && timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $O/c4_r01.json 2> $O/c4_r01.err)
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $O/c4_r02.json 2> $O/c4_r02.err
