set -x
python -m pytest tests/test_gpu_idem.py -x -q > gpurun_out/idem_tests.log 2>&1; tail -2 gpurun_out/idem_tests.log
python tools/route_once.py --config c2 --shape 4096,4096 --op max --route bdbs --box 4,4 > gpurun_out/p1.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:"k_fused_pair" -s 2 -c 1 -o gpurun_out/c3a_i64 python tools/route_once.py --config c2 --shape 4096,4096 --op max --route bdbs --box 4,4 > gpurun_out/ncu1.log 2>&1
python tools/route_once.py --config c4 --shape 4096,4096 --route bdbs --box 4,4 > gpurun_out/p2.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:"k_fused_pair" -s 2 -c 1 -o gpurun_out/c3a_f32 python tools/route_once.py --config c4 --shape 4096,4096 --route bdbs --box 4,4 > gpurun_out/ncu2.log 2>&1
python tools/route_once.py --config c2 --route box-complement --reps 3 > gpurun_out/p3.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:"k_idem" -s 2 -c 2 -o gpurun_out/c2_idem python tools/route_once.py --config c2 --route box-complement --reps 3 > gpurun_out/ncu3.log 2>&1
ls gpurun_out/*.ncu-rep
