N="ncu --set full --import-source on --clock-control none"
$N -k regex:"scan_v2|rad_sparse2" --launch-skip 6 -c 3 -o gpurun_out/r2_scan python profiles/prof_run.py c3 3 > gpurun_out/ncu_scan.log 2>&1
ncu -i gpurun_out/r2_scan.ncu-rep --page details 2>/dev/null | grep -E "^  [a-z_A-Z:<>0-9, ()]*\(|bank conflicts|excessive" | cut -c1-220
$N -k regex:"rad_gemm2s|recombine16|band3" --launch-skip 6 -c 3 -o gpurun_out/r2_c2b python profiles/prof_run.py c2 3 > gpurun_out/ncu_c2b.log 2>&1
ncu -i gpurun_out/r2_c2b.ncu-rep --page details 2>/dev/null | grep -E "^  [a-z_A-Z:<>0-9, ()]*\(|bank conflicts|excessive" | cut -c1-220
