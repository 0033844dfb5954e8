# c4 device timeline (CUPTI) and ncu --set full of the register dot kernel (source lines, pipes)
python profiles/kineto_timeline.py c4 2 > gpurun_out/timeline_c4.txt 2>&1
python profiles/kineto_timeline.py c3 3 > gpurun_out/timeline_c3.txt 2>&1
python profiles/kineto_timeline.py c2 3 > gpurun_out/timeline_c2.txt 2>&1
python profiles/prof_run.py c1 2 > /dev/null 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:dot_reg -c 1 -o gpurun_out/r2_c1 python profiles/prof_run.py c1 2 > gpurun_out/ncu_c1.log 2>&1
python profiles/ncu_summary.py gpurun_out/r2_c1.ncu-rep > gpurun_out/r2_c1.summary.txt 2>&1
python profiles/ncu_lines.py gpurun_out/r2_c1.ncu-rep 80 > gpurun_out/r2_c1.lines.txt 2>&1
ncu -i gpurun_out/r2_c1.ncu-rep --page details > gpurun_out/r2_c1.details.txt 2>&1
