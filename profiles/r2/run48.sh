for i in 1 2 3; do python profiles/e2e_only.py 1 2>&1 | tail -1; done
for i in 1 2 3; do timeout 300 python bench.py --steps 20 --warmup 5 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print(d['ms_per_step'], d['e2e']['ms_per_step'], d['e2e']['sync_call']['ms_per_step'])"; done
