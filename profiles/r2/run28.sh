for v in "" old ""; do
  if [ -n "$v" ]; then export APB_LIB_PATH=$PWD/variants/lib_oldgemm.so; else unset APB_LIB_PATH; fi
  echo "== variant '$v'"
  APB_BAND_BN=256 APB_BAND_KSPLIT=1 timeout 300 python bench.py --steps 20 --warmup 5 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print(d['ms_per_step'], d['roofline']['kernel_ms'], d['roofline']['frac'], d['also']['c4']['ms_per_step'], d['also']['c4']['roofline']['frac'])"
done
