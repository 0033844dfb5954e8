python profiles/kineto_timeline.py c3 3 2>&1 | tail -10
for v in rb4 rb16; do echo "== $v"; APB_LIB_PATH=$PWD/variants/lib_$v.so python profiles/kineto_timeline.py c3 3 2>&1 | grep -E "recombine|step span"; done
