timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; tail -3 gpurun_out/gputests.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 300 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2> gpurun_out/bench.err; tail -c 300 gpurun_out/bench.log; echo
timeout 300 python bench.py > gpurun_out/bench_default.log 2> gpurun_out/bench_default.err; python - <<'P'
import json
for f in ('gpurun_out/bench.log','gpurun_out/bench_default.log'):
    d=json.loads(open(f).read().strip().splitlines()[-1])
    print(f, d['steps'], d['ms_per_step'], d['roofline']['kernel_ms'], d['roofline']['frac'], d['e2e']['ms_per_step'], d['also']['c1']['ms_per_step'], d['also']['c2']['ms_per_step'], d['also']['c4']['ms_per_step'], d['also']['c4']['roofline']['frac'], d['gpu_launches'], d['clocks'])
P
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1; tail -c 300 gpurun_out/bench_ref.log
bash profiles/r2_capture.sh
