# Round 2, last session: ncu --set full of the small-config (C2 / C3) kernels in their final
# state; each profiled command first exits 0 without ncu.
set -x
R="python tools/route_once.py"
NCU="ncu --set full --clock-control none --import-source on"
$R --config c2 --route box-complement --reps 3 > gpurun_out/p_c2.log 2>&1 &&
$NCU -k regex:"k_idem" -s 2 -c 2 -o gpurun_out/r2s4_c2_idem $R --config c2 --route box-complement --reps 3 > gpurun_out/n_c2.log 2>&1
$R --config c4 --shape 4096,4096 --route bdbs --box 4,4 > gpurun_out/p_c3a.log 2>&1 &&
$NCU -k regex:"k_fused_pair" -s 2 -c 1 -o gpurun_out/r2s4_c3a_f32 $R --config c4 --shape 4096,4096 --route bdbs --box 4,4 > gpurun_out/n_c3a.log 2>&1
$R --config c2 --shape 4096,4096 --op max --route bdbs --box 4,4 > gpurun_out/p_c3ai.log 2>&1 &&
$NCU -k regex:"k_fused_pair" -s 2 -c 1 -o gpurun_out/r2s4_c3a_i64 $R --config c2 --shape 4096,4096 --op max --route bdbs --box 4,4 > gpurun_out/n_c3ai.log 2>&1
$R --config c4 --shape 32,32,32,32,32 --route bdbs --box 4,4,4,4,4 > gpurun_out/p_c3d.log 2>&1 &&
$NCU -k regex:"k_outer_pair|k_block" -s 2 -c 2 -o gpurun_out/r2s4_c3d_f32 $R --config c4 --shape 32,32,32,32,32 --route bdbs --box 4,4,4,4,4 > gpurun_out/n_c3d.log 2>&1
$R --config c4 --shape 16,16,16,16,16,16 --route bdbs --box 4,4,4,4,4,4 > gpurun_out/p_c3e.log 2>&1 &&
$NCU -k regex:"k_outer_pair|k_block|k_axis|k_strided" -s 3 -c 3 -o gpurun_out/r2s4_c3e_f32 $R --config c4 --shape 16,16,16,16,16,16 --route bdbs --box 4,4,4,4,4,4 > gpurun_out/n_c3e.log 2>&1
ls -la gpurun_out/*.ncu-rep
tail -2 gpurun_out/p_c3d.log gpurun_out/n_c3d.log
