python profiles/prof_run.py c1 2 > /dev/null 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:dot_reg -c 1 -o gpurun_out/r2_c1b python profiles/prof_run.py c1 2 > gpurun_out/ncu_c1.log 2>&1
python profiles/ncu_summary.py gpurun_out/r2_c1b.ncu-rep
python profiles/ncu_lines.py gpurun_out/r2_c1b.ncu-rep 45
ncu -i gpurun_out/r2_c1b.ncu-rep --page details 2>/dev/null | grep -E "Pipe|pipe|Issue Slots|Executed Ipc|L1/TEX Hit|Mem Busy|Max Bandwidth|DRAM Throughput|Eligible|No Eligible|Registers|Theoretical Occ|Achieved Occ" | head -40
