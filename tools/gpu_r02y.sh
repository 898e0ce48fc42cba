O=gpurun_out/r02y
mkdir -p $O
timeout 120 tools/probes/warp_rates > $O/warp_rates.jsonl 2>&1
