# second r1 capture: the band GEMM with accumulator normalisation (c5 p=512),
# the dense radius products and GEMM at N=2048 p=64, dot_small at p=256
N="ncu --set full --import-source on --clock-control none"
$N -k regex:"band3|recombine" -c 2 -o gpurun_out/r1_c5m python profiles/prof_run.py c5m 1 > gpurun_out/ncu_c5m.log 2>&1
$N -k regex:"band3|rad_gemm2|rad_sparse2|pack_ab|fused_planes" -c 3 -o gpurun_out/r1_c5m64 python profiles/prof_run.py c5m64 1 > gpurun_out/ncu_c5m64.log 2>&1
$N -k regex:dot_small -c 1 -o gpurun_out/r1_c5ds python profiles/prof_run.py c5ds 1 > gpurun_out/ncu_c5ds.log 2>&1
for r in r1_c5m r1_c5m64 r1_c5ds; do
  python profiles/ncu_summary.py gpurun_out/$r.ncu-rep > gpurun_out/$r.summary.txt 2>&1
  python profiles/ncu_lines.py gpurun_out/$r.ncu-rep 25 > gpurun_out/$r.lines.txt 2>&1
  rm -f gpurun_out/$r.ncu-rep
done
