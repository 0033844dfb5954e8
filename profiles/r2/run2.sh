python -m pytest tests/test_dot_gpu.py -x -q 2>&1 | tail -3
python profiles/dotbench.py c1 > gpurun_out/plain.log 2>&1 && cat gpurun_out/plain.log && ncu --set full --clock-control none --import-source on -k regex:dot_reg -s 3 -c 1 -o gpurun_out/dotreg2 python profiles/dotbench.py c1 > gpurun_out/ncu.log 2>&1; tail -1 gpurun_out/ncu.log
APB_REG_TPD=16 python profiles/dotbench.py c1
