O=gpurun_out/r02v
mkdir -p $O
timeout 120 tools/probes/potrf_trace > $O/potrf_trace.jsonl 2>&1; echo "rc=$?" >> $O/potrf_trace.jsonl
