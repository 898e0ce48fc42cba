# round 2, first GPU pass: the -m gpu suite (minus the full-size config
# parity, whose fixtures are still being generated), the C4 bench at 1 GPU,
# --gpus 2 refusal on a 1-GPU box, and the 2-rank path through the bench
set -x
mkdir -p gpurun_out/r02a
nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv > gpurun_out/r02a/gpu.txt
nproc > gpurun_out/r02a/host.txt; free -g >> gpurun_out/r02a/host.txt; lscpu | grep -E "Model name|Socket|Core|Thread" >> gpurun_out/r02a/host.txt
timeout 1500 python -m pytest tests -m gpu -x -q --deselect tests/test_gpu_configs.py -p no:cacheprovider > gpurun_out/r02a/pytest.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/r02a/pytest.txt
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/r02a/bench.json 2> gpurun_out/r02a/bench.err; echo "rc=$?" >> gpurun_out/r02a/bench.err
timeout 120 python bench.py --gpus 2 --steps 1 --warmup 1 > gpurun_out/r02a/refuse.txt 2>&1; echo "rc=$?" >> gpurun_out/r02a/refuse.txt
timeout 900 python bench.py --gpus 2 --debug-share-gpu --steps 1 --warmup 1 --e2e-steps 1 --tile 512 > gpurun_out/r02a/share2.json 2> gpurun_out/r02a/share2.err; echo "rc=$?" >> gpurun_out/r02a/share2.err
