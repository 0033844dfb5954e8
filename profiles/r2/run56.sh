python profiles/c4_real_product.py > /dev/null 2>&1 && ncu --set full --import-source on --clock-control none -k regex:rad_gemm2_kernel -c 1 -o gpurun_out/r2_radg python profiles/c4_real_product.py > gpurun_out/ncu_radg.log 2>&1
python profiles/ncu_summary.py gpurun_out/r2_radg.ncu-rep
python profiles/ncu_lines.py gpurun_out/r2_radg.ncu-rep 14
ncu -i gpurun_out/r2_radg.ncu-rep --page details 2>/dev/null | grep -E "Executed Ipc|Issue Slots|FP64|fp64|Pipe|Eligible|Theoretical Occ|Achieved Occ|Block Limit|Bank conf|bank conf" | head -20
