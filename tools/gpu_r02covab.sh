O=gpurun_out/r02covab
mkdir -p $O
for i in 1 2; do
  for v in default mb4 u4mb4 u4 u6; do
    if [ $v = default ]; then unset BGP_LIB_PATH; else export BGP_LIB_PATH=$PWD/build/var_$v/libbgp.so; fi
    timeout 300 python tools/cov_time.py 2>/dev/null | sed "s/^{/{\"v\": \"$v\", /" >> $O/cov.jsonl
  done
done
