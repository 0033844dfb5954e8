APB_RAD_NO_BESIDE=1 python profiles/kineto_timeline.py c3 3 2>&1 | tail -11
APB_RAD_NO_BESIDE=1 ncu --set full --import-source on --clock-control none -k regex:rad_quad -c 1 -o gpurun_out/r2_radquad python profiles/prof_run.py c3 2 > gpurun_out/ncu_radquad.log 2>&1
python profiles/ncu_summary.py gpurun_out/r2_radquad.ncu-rep
python profiles/ncu_lines.py gpurun_out/r2_radquad.ncu-rep 30
