timeout 900 python -m pytest tests/test_matmul_gpu.py -m gpu -x -q -k "golden or full_config or repeated or replay" > gpurun_out/gputests_mm.log 2>&1; tail -2 gpurun_out/gputests_mm.log
for w in 4 3 2 0; do echo "== wave $w"; APB_PACK_WAVE=$w python profiles/kineto_timeline.py c3 3 2>&1 | grep -E "span|pack_ab|rad_sparse2|band3"; done
