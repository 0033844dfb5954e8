timeout 900 python -m pytest tests/test_dot_gpu.py tests/test_fuzz_gpu.py tests/test_poly_gpu.py -m gpu -x -q > gpurun_out/gputests_dot.log 2>&1; tail -12 gpurun_out/gputests_dot.log
timeout 300 python profiles/dotbench.py c1 2>&1 | tail -3
APB_REG_NOTAIL=1 timeout 300 python profiles/dotbench.py c1 2>&1 | tail -3
