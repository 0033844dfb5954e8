timeout 1200 python -m pytest tests/test_matmul_gpu.py -m gpu -x -q -k "centred or replay or repeated or golden or full_config" > gpurun_out/gputests_mm.log 2>&1; tail -2 gpurun_out/gputests_mm.log
timeout 300 python bench.py --steps 20 --warmup 5 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print(d['ms_per_step'], d['e2e']['ms_per_step'], d['also']['c2']['ms_per_step'], d['also']['c4']['ms_per_step'])"
