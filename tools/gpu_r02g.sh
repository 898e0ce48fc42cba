# pipelined C2: SMs each lane leaves to the other (0, 4, 8, 16)
set -x
O=gpurun_out/r02g
mkdir -p $O
for r in 0 4 8 16; do BGP_LANE_RESERVE=$r timeout 600 python tools/bench_configs.py --configs 2 --tile 256 > $O/c2_res$r.jsonl 2> $O/c2_res$r.err; done
