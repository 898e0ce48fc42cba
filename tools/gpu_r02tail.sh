O=gpurun_out/r02tail
mkdir -p $O
for tl in 8 12 16 24 32; do BGP_TAIL=$tl timeout 600 python tools/bench_configs.py --configs 2,3 --tile 512 2>/dev/null | sed "s/^{/{\"tail\": $tl, /" >> $O/tail512.jsonl; done
for tl in 24 32 48; do BGP_TAIL=$tl timeout 600 python tools/bench_configs.py --configs 2,3 --tile 256 2>/dev/null | sed "s/^{/{\"tail\": $tl, /" >> $O/tail256.jsonl; done
