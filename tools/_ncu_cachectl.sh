set -x
R="python tools/route_once.py"
NCU="ncu --cache-control none --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct"
$NCU -k regex:"k_outer_pair|k_block|k_axis|k_strided|k_fused" -s 6 -c 6 --csv --log-file gpurun_out/cc_c3e.csv $R --config c4 --shape 16,16,16,16,16,16 --route bdbs --box 4,4,4,4,4,4 --reps 4 > gpurun_out/cc1.log 2>&1
$NCU -k regex:"k_outer_pair|k_block|k_axis|k_strided|k_fused" -s 4 -c 4 --csv --log-file gpurun_out/cc_c3b.csv $R --config c4 --shape 256,256,256 --route bdbs --box 4,4,4 --reps 4 > gpurun_out/cc2.log 2>&1
$NCU -k regex:"k_outer_pair|k_block|k_axis|k_strided|k_fused" -s 4 -c 4 --csv --log-file gpurun_out/cc_c3c.csv $R --config c4 --shape 64,64,64,64 --route bdbs --box 4,4,4,4 --reps 4 > gpurun_out/cc3.log 2>&1
