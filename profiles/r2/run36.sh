timeout 1500 python profiles/run_configs.py c4 c5 > gpurun_out/configs_c4_c5.log 2>&1; grep -o '"c[45][_p0-9]*": {"ms": [0-9.]*' gpurun_out/configs_c4_c5.log; grep -c '"bit_identical": true' gpurun_out/configs_c4_c5.log
timeout 600 python profiles/dotbench.py c5 > gpurun_out/dots_c5.log 2>&1; tail -12 gpurun_out/dots_c5.log
python profiles/kineto_timeline.py c4 2 2>&1 | grep -v arn > gpurun_out/timeline_c4.txt
python profiles/kineto_timeline.py c2 3 2>&1 | grep -v arn > gpurun_out/timeline_c2.txt
python profiles/kineto_timeline.py c3 3 2>&1 | grep -v arn > gpurun_out/timeline_c3.txt
