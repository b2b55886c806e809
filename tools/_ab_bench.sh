# A/B of the headline bench line: balanced unit ranges of the fused pair on / off, alternated
for i in 1 2 3; do
  for b in 1 0; do
    EXSUM_FP_BALANCED=$b python bench.py --no-e2e --no-cpu --steps 20 --warmup 3 | python -c "
import sys, json
d = json.loads(sys.stdin.read()); k = d['kernels']
print('balanced=$b step %.4f ms  axis %.4f  pair %.4f  bdbsc %.4f bdbs %.4f' % (d['ms_per_step'], k['pass_strided[8192MiB]']['avg_ms'], k['fused_pair[8196MiB]']['avg_ms'], d['routes']['bdbsc']['ms_per_step'], d['routes']['bdbs']['ms_per_step']))"
  done
done
