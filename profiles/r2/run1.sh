set -x
python -m pytest tests/test_dot_gpu.py -x -q 2>&1 | tail -15
python profiles/dotbench.py c1
APB_REG_TPD=16 python profiles/dotbench.py c1
APB_DOT_NOREG=1 python profiles/dotbench.py c1
