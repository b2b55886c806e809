set -x
python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/plain_bench.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches_bench_c4.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_l.log 2>&1
python tools/route_once.py --config c4 --route box-complement --reps 2 > gpurun_out/plain_c4.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:"k_fused_pair|k_axis_stream|k_tail" -s 4 -c 4 -o gpurun_out/r2_c4_final python tools/route_once.py --config c4 --route box-complement --reps 2 > gpurun_out/ncu_c4.log 2>&1
python tools/route_once.py --config c2 --route box-complement --reps 3 > gpurun_out/plain_c2.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:"k_idem" -s 2 -c 2 -o gpurun_out/r2_c2_final python tools/route_once.py --config c2 --route box-complement --reps 3 > gpurun_out/ncu_c2.log 2>&1
ls -la gpurun_out | tail -5
