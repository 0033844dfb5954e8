ncu --set full --import-source on --clock-control none -k regex:rad_tile -c 1 -o gpurun_out/r2_radtile python profiles/prof_run.py c3 2 > gpurun_out/ncu_radtile.log 2>&1
python profiles/ncu_summary.py gpurun_out/r2_radtile.ncu-rep
python profiles/ncu_lines.py gpurun_out/r2_radtile.ncu-rep 40
