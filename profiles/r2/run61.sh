timeout 1500 python -m pytest tests/test_matmul_gpu.py tests/test_fuzz_gpu.py -m gpu -x -q > gpurun_out/gputests_mm.log 2>&1; tail -2 gpurun_out/gputests_mm.log
python profiles/kineto_timeline.py c3 3 2>&1 | grep -E "pack_ab|rad_sparse|band3|span"
APB_PACK_A1=1 python profiles/kineto_timeline.py c3 3 2>&1 | grep -E "pack_ab|rad_sparse|band3|span"
python profiles/kineto_timeline.py c4 2 2>&1 | grep -E "pack_ab|span" | head -2
timeout 300 python bench.py --steps 20 --warmup 5 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print(d['ms_per_step'], d['e2e']['ms_per_step'], d['also']['c2']['ms_per_step'], d['also']['c4']['ms_per_step'])"
