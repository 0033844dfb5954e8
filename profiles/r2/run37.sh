cat > /tmp/p1024.py <<'P'
import sys, os
sys.path.insert(0, os.getcwd())
import torch
from paper_1901_04289_b200 import gen, ops
import ctypes as C
for p, n in ((1024, 2048), (512, 2048)):
    a, b = gen.config5_matrices(n=n, p=p)
    A, B = ops.BallMatrix(a.to_device(), n, n), ops.BallMatrix(b.to_device(), n, n)
    lib = ops._lib.lib()
    out = ops.block_matmul_ball(A, B, p)
    ts = []
    for _ in range(3):
        lib.apb_gemm_timer_reset()
        s, e = torch.cuda.Event(True), torch.cuda.Event(True)
        s.record(); ops.block_matmul_ball(A, B, p, out=out); e.record(); torch.cuda.synchronize()
        g, l = C.c_uint64(0), C.c_uint64(0); lib.apb_gemm_timer_read(C.byref(g), C.byref(l))
        ts.append((round(s.elapsed_time(e), 2), round(g.value / 1e6, 2)))
    print(p, n, ts, flush=True)
P
for v in "" r2start ""; do
  if [ -n "$v" ]; then export APB_LIB_PATH=$PWD/variants/lib_$v.so; else unset APB_LIB_PATH; fi
  echo "== variant '$v'"; python /tmp/p1024.py 2>&1 | tail -2
done
