# r2 session 4 baseline: timelines, band GEMM clock trace, launch list and ncu --set full of the c3 step
python profiles/kineto_timeline.py c3 3 > gpurun_out/timeline_c3.txt 2>&1
python profiles/kineto_timeline.py c2 3 > gpurun_out/timeline_c2.txt 2>&1
APB_GEMM_DEBUG=4 python profiles/prof_run.py c3 2 > gpurun_out/gemm_trace_c3.txt 2>&1
python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2> gpurun_out/bench.err; tail -c 600 gpurun_out/bench.log
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_bench_c3.csv python bench.py --steps 3 --warmup 3 > gpurun_out/ncu_bench.log 2>&1
python profiles/prof_run.py c3 3 > /dev/null 2>&1 && \
ncu --set full --import-source on --clock-control none --launch-skip 18 -c 9 -o gpurun_out/r2_c3 python profiles/prof_run.py c3 3 > gpurun_out/ncu_c3.log 2>&1
python profiles/ncu_summary.py gpurun_out/r2_c3.ncu-rep > gpurun_out/r2_c3.summary.txt 2>&1
cat gpurun_out/r2_c3.summary.txt | head -40
