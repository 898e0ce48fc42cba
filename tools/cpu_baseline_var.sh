mkdir -p gpurun_out/cpuv
nproc > gpurun_out/cpuv/info.txt; lscpu | grep -E "Model name|Socket|Core|Thread|NUMA" >> gpurun_out/cpuv/info.txt
for i in 1 2; do timeout 300 python bench.py --impl reference --steps 1 --warmup 1 > gpurun_out/cpuv/ref_$i.json 2>&1; done
timeout 300 python -c "
import sys, json; sys.path.insert(0, '.')
import bench
X, y, sc = bench.load_c4()
for i in range(2):
    r = bench.cpu_reference(10, X); print(json.dumps({'evals_per_s': r['evals_per_s'], 'chol_tflops': r['chol_tflops']}))
" > gpurun_out/cpuv/bench_sampler.txt 2>&1
