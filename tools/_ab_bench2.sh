# A/B of the headline bench line: balanced tail of the axis pass on / off (and the grid-strided uniform part), alternated
run() { python bench.py --no-e2e --no-cpu --steps 20 --warmup 3 | python -c "
import sys, json
d = json.loads(sys.stdin.read()); k = d['kernels']
print('$1 step %.4f ms  axis %.4f  pair %.4f  bdbsc %.4f bdbs %.4f' % (d['ms_per_step'], k['pass_strided[8192MiB]']['avg_ms'], k['fused_pair[8196MiB]']['avg_ms'], d['routes']['bdbsc']['ms_per_step'], d['routes']['bdbs']['ms_per_step']))"; }
for i in 1 2 3; do
  EXSUM_AS_BAL_TAIL=1 run "tail=1     "
  EXSUM_AS_BAL_TAIL=0 run "tail=0     "
  EXSUM_LIB=$PWD/variants/as_gu4.so run "tail=1 gu4 "
done
