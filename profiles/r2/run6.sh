python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; tail -5 gpurun_out/gputests.log
python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2> gpurun_out/bench.err; tail -c 3000 gpurun_out/bench.log
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1; cat gpurun_out/bench_ref.log
