for v in "" s5p5 s6p5 s6p6 s8p6; do
  if [ -n "$v" ]; then export APB_LIB_PATH=$PWD/variants/lib_$v.so; else unset APB_LIB_PATH; fi
  echo "== variant '$v'"; python profiles/kineto_timeline.py c3 3 2>&1 | grep -E "span|scan_v2_kernel|pack_ab|band3"
done
unset APB_LIB_PATH
python profiles/kineto_timeline.py c4 2 2>&1 | grep -v arn > gpurun_out/timeline_c4.txt; head -40 gpurun_out/timeline_c4.txt
timeout 1500 python profiles/run_configs.py c4 c5 > gpurun_out/configs_c4_c5.log 2>&1; tail -c 1500 gpurun_out/configs_c4_c5.log
