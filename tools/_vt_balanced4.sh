V="variants/fp_notail.so"
for spec in "c5 bdbs add 512,512,512 2,2,2" "c5 bdbs add 512,512,512 4,4,4" "c5 bdbsc add 512,512,512 2,2,2" "c4 bdbs add 1024,1024,1024 2,2,2" "c4 bdbs add 1024,1024,1024 4,4,4" "c4 bdbsc add 1024,1024,1024 4,4,4" "c5 bdbs add 300,512,512 4,4,4"; do
  set -- $spec
  echo "== $spec"
  python tools/variant_time.py --config $1 --route $2 --op $3 --shape $4 --box $5 --reps 10 $V | python -c "
import sys, json
for l in sys.stdin:
    n, j = l.split(' ', 1); d = json.loads(j); print('  %-14s step %.4f fused_pair %.4f' % (n, d['step_ms'], d['kernels'].get('fused_pair', 0)))"
done
