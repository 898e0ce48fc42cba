# per-step C5 profile: round-1 tree vs current
set -x
O=$PWD/gpurun_out/r02o
mkdir -p $O
(cd build/r01_tree && timeout 600 python tools/step_profile_c5.py > $O/steps_r01.json 2> $O/steps_r01.err)
timeout 600 python tools/step_profile_c5.py > $O/steps_r02.json 2> $O/steps_r02.err
