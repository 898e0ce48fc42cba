O=gpurun_out/r02x
mkdir -p $O
timeout 120 tools/probes/chol32_variants > $O/chol32.jsonl 2>&1
