for d in 0 2 4 8; do echo "== rad debug $d"; APB_RAD_DEBUG=$d python profiles/kineto_timeline.py c3 3 2>&1 | grep -E "band3|rad_quad|step span"; done
