python - <<'PY'
import sys, os, torch
sys.path.insert(0, os.getcwd())
from paper_1901_04289_b200 import gen, ops
x, y = gen.config1_dots()
dx, dy = x.to_device(), y.to_device()
from paper_1901_04289_b200.balls import DeviceBallArray
out = DeviceBallArray.empty(65536, 2)
for _ in range(3): ops.dot_batch(dx, dy, 100, 65536, 128, out=out)
torch.cuda.synchronize()
s, e = torch.cuda.Event(True), torch.cuda.Event(True)
s.record()
for _ in range(10): ops.dot_batch(dx, dy, 100, 65536, 128, out=out, check=False)
e.record(); torch.cuda.synchronize()
print("dot ms", s.elapsed_time(e)/10, os.environ.get("APB_DOT_RELOAD"))
PY
