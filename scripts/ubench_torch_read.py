import torch, time
for k in (11, 22, 33, 66):
    x = torch.randn(k, 8_000_000, device='cuda', dtype=torch.float64)
    for _ in range(3): y = x.sum(dim=1)
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(10): y = x.sum(dim=1)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"torch sum rows k={k}: {ms*1e3:.1f} us  {k*8e6*8/ms/1e6:.0f} GB/s")
    xt = x.t().contiguous()  # row-major n x k
    for _ in range(3): y = xt.sum(dim=0)
    e0.record()
    for _ in range(10): y = xt.sum(dim=0)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"torch sum (n,k) rowmajor k={k}: {ms*1e3:.1f} us  {k*8e6*8/ms/1e6:.0f} GB/s")
    del x, xt
