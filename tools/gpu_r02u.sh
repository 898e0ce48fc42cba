set -x
O=gpurun_out/r02u
mkdir -p $O
timeout 600 python tools/step_profile.py --config 4 --tile 512 > $O/steps_c4_512.json 2> $O/steps_c4.err
timeout 600 python tools/step_profile.py --config 2 --tile 256 > $O/steps_c2_256.json 2> $O/steps_c2.err
timeout 600 python tools/step_profile.py --config 2 --tile 128 > $O/steps_c2_128.json 2> $O/steps_c2_128.err
timeout 600 ncu --set full --clock-control none -k regex:gemm_dmma --launch-skip 2 -c 1 -o $O/c2_step2 -f python tools/step_profile.py --config 2 --tile 256 > $O/ncu1.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:gemm_dmma --launch-skip 30 -c 1 -o $O/c2_step30 -f python tools/step_profile.py --config 2 --tile 256 > $O/ncu2.log 2>&1
