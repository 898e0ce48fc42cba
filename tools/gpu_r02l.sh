# A/B: which round-2 GEMM change costs C5 ~1 %
set -x
O=$PWD/gpurun_out/r02l
mkdir -p $O
for v in prod r01 OLD_ROLE NO_TMT NO_PAD prod r01; do
  if [ $v = r01 ]; then
    (cd build/r01_tree && timeout 600 python tools/bench_configs.py --configs 5 --tile 512 >> $O/c5_$v.jsonl 2>> $O/c5_$v.err)
  elif [ $v = prod ]; then
    timeout 600 python tools/bench_configs.py --configs 5 --tile 512 >> $O/c5_$v.jsonl 2>> $O/c5_$v.err
  else
    BGP_LIB_PATH=$PWD/build/ab_$v/libbgp.so timeout 600 python tools/bench_configs.py --configs 5 --tile 512 >> $O/c5_$v.jsonl 2>> $O/c5_$v.err
  fi
done
