# A/B of producer variants on the C5 step profile
set -x
O=$PWD/gpurun_out/r02p
mkdir -p $O
for v in prod p64 claim claim_p64 prod r01; do
  if [ $v = r01 ]; then (cd build/r01_tree && timeout 600 python tools/step_profile_c5.py > $O/steps_$v.json 2> $O/steps_$v.err)
  elif [ $v = prod ]; then timeout 600 python tools/step_profile_c5.py >> $O/steps_$v.json 2>> $O/steps_$v.err
  else BGP_LIB_PATH=$PWD/build/ab_$v/libbgp.so timeout 600 python tools/step_profile_c5.py > $O/steps_$v.json 2> $O/steps_$v.err; fi
done
