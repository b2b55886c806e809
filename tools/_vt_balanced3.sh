V="variants/bal_pct0.so"
for spec in "c5 bdbs add 512,512,512 4,4,4" "c5 box-complement add 512,512,512 2,2,2" "c5 box-complement add 512,512,512 4,4,4" "c4 bdbs add 1024,1024,1024 2,2,2" "c4 bdbs add 1024,1024,1024 4,4,4" "c4 bdbs add 1024,1024,1024 8,8,8" "c4 box-complement add 1024,1024,1024 4,4,4" "c4 box-complement add 1024,1024,1024 8,8,8" "c4 bdbs add 128,1024,1024 2,2,2" "c4 bdbs add 128,1024,1024 4,4,4" "c4 bdbsc add 1024,1024,1024 16,16,16"; do
  set -- $spec
  echo "== $spec"
  python tools/variant_time.py --config $1 --route $2 --op $3 --shape $4 --box $5 --reps 10 $V | python -c "
import sys, json
for l in sys.stdin:
    n, j = l.split(' ', 1); d = json.loads(j); print('  %-12s step %.4f fused_pair %.4f' % (n, d['step_ms'], d['kernels'].get('fused_pair', 0)))"
  EXSUM_FP_BALANCED=0 python tools/variant_time.py --config $1 --route $2 --op $3 --shape $4 --box $5 --reps 10 | python -c "
import sys, json
for l in sys.stdin:
    n, j = l.split(' ', 1); d = json.loads(j); print('  %-12s step %.4f fused_pair %.4f' % ('uniform', d['step_ms'], d['kernels'].get('fused_pair', 0)))"
done
