V="variants/nostripbal.so"
for spec in "c4 bdbs add 64,2048,2048 16,16,16" "c4 bdbs add 64,2048,2048 8,8,8" "c4 bdbs add 64,2048,2048 4,4,4" "c4 bdbs add 16,4096,4096 16,16,16" "c5 bdbs add 32,2048,2048 8,8,8" "c4 bdbs add 8192,8192 16,16" "c4 bdbs add 4096,4096 16,16"; do
  set -- $spec
  echo "== $spec"
  python tools/variant_time.py --config $1 --route $2 --op $3 --shape $4 --box $5 --reps 10 $V | python -c "
import sys, json
for l in sys.stdin:
    n, j = l.split(' ', 1); d = json.loads(j); print('  %-14s step %.4f  %s' % (n, d['step_ms'], {k: round(v, 4) for k, v in d['kernels'].items()}))"
done
