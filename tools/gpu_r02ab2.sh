# A/B: HEAD build vs working tree, C4 bench (2x each, alternating) + C1/C2
O=${1:-gpurun_out/ab2}
mkdir -p $O
for i in 1 2; do
  for v in head new; do
    if [ $v = head ]; then export BGP_LIB_PATH=$PWD/build/ab/libbgp_head.so; else unset BGP_LIB_PATH; fi
    timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 2>/dev/null | tail -1 | sed "s/^{/{\"build\": \"$v\", /" >> $O/c4.jsonl
    timeout 600 python tools/bench_configs.py --configs 1,2 --tile 256 2>/dev/null | sed "s/^{/{\"build\": \"$v\", /" >> $O/c12.jsonl
  done
done
