# ablation driver: kernel_report for each build/var/$VARS.so (tools/build_variant.sh) over $CFGS
for v in $VARS; do echo "== $v"; EXSUM_LIB=build/var/$v.so python tools/kernel_report.py --configs $CFGS --reps 5 | python -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: continue
    print(d['config'],d['route'],d['op'],d['box'],d['step_ms'], [(k,round(v['ms'],4),v['frac']) for k,v in d['kernels'].items() if v['ms']>0.02])
"; done
