for g in 1 37 74 148; do echo "== rad grid $g"; APB_RAD_GRID=$g python profiles/kineto_timeline.py c3 3 2>&1 | grep -E "band3|rad_quad|step span"; done
