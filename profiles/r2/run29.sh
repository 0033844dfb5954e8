python profiles/kineto_timeline.py c3 3 2>&1 | tail -10
APB_RAW32=1 python profiles/kineto_timeline.py c3 3 2>&1 | grep -E "band3|recombine|span"
