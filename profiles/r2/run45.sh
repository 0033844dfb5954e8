timeout 900 python -m pytest tests/test_matmul_gpu.py -m gpu -x -q -k "golden or full_config or repeated or replay or PACK" > gpurun_out/gputests_mm.log 2>&1; tail -2 gpurun_out/gputests_mm.log
python profiles/kineto_timeline.py c3 3 2>&1 | grep -v arn | tail -9
python profiles/kineto_timeline.py c2 3 2>&1 | grep -v arn | tail -9
timeout 300 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2> gpurun_out/bench.err; python - <<'P'
import json
d=json.loads(open('gpurun_out/bench.log').read().strip().splitlines()[-1])
print(d['ms_per_step'], d['roofline']['kernel_ms'], d['roofline']['frac'], d['e2e']['ms_per_step'], d['also']['c2']['ms_per_step'], d['also']['c2']['roofline']['kernel_ms'], d['also']['c4']['ms_per_step'], d['also']['c4']['roofline']['frac'])
P
