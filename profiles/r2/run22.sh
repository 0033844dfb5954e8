APB_RAD_NO_BESIDE=1 python profiles/kineto_timeline.py c3 3 2>&1 | tail -10
