for v in "" ru1 ru8; do
  if [ -n "$v" ]; then export APB_LIB_PATH=$PWD/variants/lib_$v.so; else unset APB_LIB_PATH; fi
  echo "== variant '$v'"
  python profiles/kineto_timeline.py c2 3 2>&1 | grep -E "span|rad_gemm2"
  python profiles/kineto_timeline.py c4 2 2>&1 | grep -E "rad_gemm2" | head -2
done
