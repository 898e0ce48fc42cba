# A/B of two builds of libbgp.so in one box: $1 = output dir
O=${1:-gpurun_out/ab}
mkdir -p $O
for i in 1 2 3; do
  for v in head new; do
    if [ $v = head ]; then export BGP_LIB_PATH=$PWD/build/ab/libbgp_head.so; else unset BGP_LIB_PATH; fi
    timeout 600 python tools/bench_configs.py --configs 1,2 --tile 128 2>/dev/null | sed "s/^{/{\"build\": \"$v\", \"tile_arg\": 128, /" >> $O/ab.jsonl
    timeout 600 python tools/bench_configs.py --configs 1 --tile 256 2>/dev/null | sed "s/^{/{\"build\": \"$v\", \"tile_arg\": 256, /" >> $O/ab.jsonl
  done
done
