set -x
N="ncu --set full --import-source on --clock-control none"
$N -c 10 -o gpurun_out/r1_c3 python profiles/prof_run.py c3 1 > gpurun_out/ncu_c3.log 2>&1
$N -k regex:dot_grp -c 1 -o gpurun_out/r1_c1 python profiles/prof_run.py c1 1 > gpurun_out/ncu_c1.log 2>&1
$N -k regex:dot_wide -c 2 -o gpurun_out/r1_c5d python profiles/prof_run.py c5d 1 > gpurun_out/ncu_c5d.log 2>&1
$N -k regex:"slice_gemm|recombine|rad_" -c 4 -o gpurun_out/r1_c5m python profiles/prof_run.py c5m 1 > gpurun_out/ncu_c5m.log 2>&1
$N -k regex:imad -c 1 -o gpurun_out/r1_imad python profiles/prof_run.py imad 1 > gpurun_out/ncu_imad.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench_c3.csv python bench.py --steps 2 --warmup 3 --no-also > gpurun_out/ncu_launch.log 2>&1
timeout 900 python profiles/run_configs.py c4 c5 > gpurun_out/configs45.log 2>&1
# text summaries on the box (the reports themselves are too large to bring back)
for r in r1_c3 r1_c1 r1_c5d r1_c5m r1_imad; do
  python profiles/ncu_summary.py gpurun_out/$r.ncu-rep > gpurun_out/$r.summary.txt 2>&1
  python profiles/ncu_lines.py gpurun_out/$r.ncu-rep 25 > gpurun_out/$r.lines.txt 2>&1
done
rm -f gpurun_out/r1_c1.ncu-rep gpurun_out/r1_c5d.ncu-rep gpurun_out/r1_c5m.ncu-rep gpurun_out/r1_imad.ncu-rep
