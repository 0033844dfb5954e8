echo "== rolled"; APB_LIB_PATH=$PWD/variants/lib_rq_rolled.so python profiles/kineto_timeline.py c3 3 2>&1 | grep -E "band3|rad_quad|step span"
echo "== rolled, standalone grid 148"; APB_RAD_GRID=148 APB_RAD_NO_BESIDE=1 APB_LIB_PATH=$PWD/variants/lib_rq_rolled.so python profiles/kineto_timeline.py c3 3 2>&1 | grep -E "rad_quad"
