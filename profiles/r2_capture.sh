# round-2 captures at HEAD: device timelines, launch list of the bench command, ncu --set full of
# the config-3 / config-2 / config-4-shaped steps and the config-1 dot kernel (each program has
# exited 0 without ncu first: the full GPU suite and the bench ran before this script)
N="ncu --set full --import-source on --clock-control none"
for c in c3 c2 c4; do python profiles/kineto_timeline.py $c 3 2>&1 | grep -v Warn | grep -v warn > gpurun_out/timeline_$c.txt; done
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_bench_c3.csv python bench.py --steps 3 --warmup 3 > gpurun_out/ncu_bench.log 2>&1
$N --launch-skip 16 -c 8 -o gpurun_out/r2_c3 python profiles/prof_run.py c3 3 > gpurun_out/ncu_c3.log 2>&1
$N --launch-skip 16 -c 8 -o gpurun_out/r2_c2 python profiles/prof_run.py c2 3 > gpurun_out/ncu_c2.log 2>&1
$N -k regex:"band3|recombine" -c 2 -o gpurun_out/r2_c5m python profiles/prof_run.py c5m 1 > gpurun_out/ncu_c5m.log 2>&1
$N -k regex:dot_reg -c 1 -o gpurun_out/r2_c1 python profiles/prof_run.py c1 2 > gpurun_out/ncu_c1.log 2>&1
for r in r2_c3 r2_c2 r2_c5m r2_c1; do
  python profiles/ncu_summary.py gpurun_out/$r.ncu-rep > gpurun_out/$r.summary.txt 2>&1
  python profiles/ncu_lines.py gpurun_out/$r.ncu-rep 30 > gpurun_out/$r.lines.txt 2>&1
done
ncu -i gpurun_out/r2_c3.ncu-rep --page details 2>/dev/null | grep -E "band3_gemm|recombine16|Tensor|tensor|Executed Ipc|DRAM Throughput|L2 Cache Throughput|Registers Per|Theoretical Occ|Achieved Occ" > gpurun_out/r2_c3.details.txt
rm -f gpurun_out/r2_c2.ncu-rep gpurun_out/r2_c5m.ncu-rep gpurun_out/r2_c1.ncu-rep
tail -20 gpurun_out/r2_c3.summary.txt
