# final-tree validation: full GPU suite, smoke, 2 ranks sharing the GPU through bench.py (tile 256, the N>1 default)
O=gpurun_out/r02check
mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "smoke rc=$?" >> $O/smoke.txt
timeout 1500 python bench.py --gpus 2 --debug-share-gpu --steps 1 --warmup 3 --e2e-steps 1 > $O/share2.json 2> $O/share2.err; echo "rc=$?" >> $O/share2.err
