for v in "" "APB_REG_TPD=16" "APB_REG_PF=1" "APB_DOT_NOREG=1"; do echo "== $v"; env $v python profiles/dotbench.py c1 2>&1 | tail -1; done
