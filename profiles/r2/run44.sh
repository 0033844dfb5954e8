python profiles/kineto_timeline.py c3 3 2>&1 | grep -v arn | tail -9
python profiles/kineto_timeline.py c2 3 2>&1 | grep -v arn | tail -9
