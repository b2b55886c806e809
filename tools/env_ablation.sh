# kernel_report for $CFGS under each environment setting in $ENVS ("A=1 B=2;A=0")
IFS=';' read -ra SETS <<< "$ENVS"
for e in "${SETS[@]}"; do echo "== $e"; env $e python tools/kernel_report.py --configs $CFGS --reps 5 | python -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: continue
    print(d['config'],d['route'],d['op'],d['box'],d['step_ms'], [(k,round(v['ms'],4),v['frac']) for k,v in d['kernels'].items() if v['ms']>0.02])
"; done
