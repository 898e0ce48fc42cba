O=gpurun_out/r02tail4
mkdir -p $O
for tl in 16 24 32 40; do BGP_TAIL=$tl timeout 600 python tools/step_profile.py --config 4 --tile 512 2>/dev/null | python -c "
import sys,json; d=json.loads(sys.stdin.read()); print(json.dumps({'tail': $tl, 'cholesky_ms': d['cholesky_ms'], 'eval_ms_wall': d['eval_ms_wall'], 'steps_sum_ms': sum(s['ms'] for s in d['steps'])}))" >> $O/c4_tail.jsonl; done
