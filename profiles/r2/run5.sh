python profiles/dotbench.py c1
APB_LIB_PATH=$PWD/variants/lib_reg_mb5.so python profiles/dotbench.py c1
APB_LIB_PATH=$PWD/variants/lib_reg_mb5.so python -m pytest tests/test_dot_gpu.py -x -q -k "golden or c1_full or edge" 2>&1 | tail -2
