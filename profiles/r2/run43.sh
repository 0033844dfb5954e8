timeout 1500 python -m pytest tests/test_matmul_gpu.py tests/test_fuzz_gpu.py -m gpu -x -q > gpurun_out/gputests_mm.log 2>&1; tail -3 gpurun_out/gputests_mm.log
python profiles/kineto_timeline.py c3 3 2>&1 | grep -v arn | tail -9
APB_NO_EARLY_PACK=1 python profiles/kineto_timeline.py c3 3 2>&1 | grep -v arn | tail -9
timeout 300 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2> gpurun_out/bench.err; python - <<'P'
import json
d=json.loads(open('gpurun_out/bench.log').read().strip().splitlines()[-1])
print(d['ms_per_step'], d['roofline']['kernel_ms'], d['roofline']['frac'], d['e2e']['ms_per_step'], d['also']['c2']['ms_per_step'], d['also']['c2']['roofline']['kernel_ms'], d['also']['c4']['ms_per_step'], d['also']['c4']['roofline']['frac'])
P
