timeout 900 python -m pytest tests/test_matmul_gpu.py -m gpu -x -q -k "golden or full_config or repeated or replay" > gpurun_out/gputests_mm.log 2>&1; tail -2 gpurun_out/gputests_mm.log
python profiles/kineto_timeline.py c3 3 2>&1 | grep -v arn | tail -9
