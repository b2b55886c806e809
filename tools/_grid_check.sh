# grids of the streaming kernels with the balanced schedules forced (2) and by the cost model (default)
for mode in 2 1; do
  for spec in "130,200,1024 16,2,4" "37,300,1024 16,16,16"; do
    set -- $spec
    EXSUM_FP_BALANCED=$mode EXSUM_AS_BAL_TAIL=$mode ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"k_fused_pair|k_axis_stream" -c 3 python tools/route_once.py --config c4 --shape $1 --route bdbs --box $2 --reps 1 2>/dev/null | python -c "
import csv, sys
rows = [r for r in csv.reader(l for l in sys.stdin if l.startswith('\"'))]
i = {k: j for j, k in enumerate(rows[0])}
for r in rows[1:]:
    print('mode $mode shape $1 box $2:', r[i['Kernel Name']][:44], 'grid', r[i['Grid Size']])"
  done
done
