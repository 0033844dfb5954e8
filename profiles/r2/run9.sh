# raw epilogue: parity on matmul tests, trace, bench
python -m pytest tests/test_matmul_gpu.py tests/test_fuzz_gpu.py -m gpu -x -q > gpurun_out/gputests_mm.log 2>&1; tail -3 gpurun_out/gputests_mm.log
APB_GEMM_DEBUG=4 python profiles/prof_run.py c3 2 2>&1 | tail -150 | head -60 > gpurun_out/gemm_trace_c3_raw.txt
python profiles/kineto_timeline.py c3 3 2>&1 | tail -10
python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2> gpurun_out/bench.err; python - <<'P'
import json
d=json.loads(open('gpurun_out/bench.log').read().strip().splitlines()[-1])
print(d['ms_per_step'], d['roofline']['kernel_ms'], d['roofline']['frac'], d['e2e']['ms_per_step'], d['also']['c2']['ms_per_step'], d['also']['c4']['ms_per_step'], d['also']['c4']['roofline']['frac'])
P
