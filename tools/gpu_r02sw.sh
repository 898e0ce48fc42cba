O=${1:-gpurun_out/r02sw}
mkdir -p $O
for i in 1 2 3; do
  for v in nosw sw; do
    unset BGP_LIB_PATH
    if [ $v = nosw ]; then export BGP_LIB_PATH=$PWD/build/ab/libbgp_nosw.so; fi
    timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 2>/dev/null | tail -1 | sed "s/^{/{\"v\": \"$v\", /" >> $O/c4.jsonl
  done
done
unset BGP_LIB_PATH
timeout 900 ncu --set full --clock-control none -k regex:gemm_dmma --launch-skip 25 -c 1 -o $O/gemm_full -f python tools/profile_c4.py --evals 0 > $O/ncu.log 2>&1; echo "ncu rc=$?" >> $O/ncu.log
