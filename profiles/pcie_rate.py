import torch, time
n = 28 << 20
h_in = torch.empty(n, dtype=torch.uint8).pin_memory(); d_in = torch.empty(n, dtype=torch.uint8, device='cuda')
h_out = torch.empty(14 << 20, dtype=torch.uint8).pin_memory(); d_out = torch.empty(14 << 20, dtype=torch.uint8, device='cuda')
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for mode in ("h2d", "d2h", "both"):
    for rep in range(3):
        torch.cuda.synchronize(); t = time.perf_counter()
        for _ in range(20):
            if mode in ("h2d", "both"):
                with torch.cuda.stream(s1): d_in.copy_(h_in, non_blocking=True)
            if mode in ("d2h", "both"):
                with torch.cuda.stream(s2): h_out.copy_(d_out, non_blocking=True)
        torch.cuda.synchronize(); dt = (time.perf_counter() - t) / 20
    print(mode, f"{dt*1e3:.3f} ms/iter", f"h2d {n/dt/1e9 if mode!='d2h' else 0:.1f} GB/s", f"d2h {(14<<20)/dt/1e9 if mode!='h2d' else 0:.1f} GB/s")
