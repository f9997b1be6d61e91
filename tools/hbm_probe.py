import torch
x = torch.empty(2*1024**3//2, dtype=torch.bfloat16, device='cuda')
y = torch.empty_like(x)
def t(fn, n=10):
    fn(); torch.cuda.synchronize()
    a,b=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n): fn()
    b.record(); torch.cuda.synchronize(); return a.elapsed_time(b)/n
ms=t(lambda: x.zero_()); print("fill (write only) GB/s", 2*1024**3/ms/1e6)
ms=t(lambda: x.fill_(1.5)); print("fill 1.5 GB/s", 2*1024**3/ms/1e6)
ms=t(lambda: y.copy_(x)); print("copy (r+w) GB/s", 2*2*1024**3/ms/1e6)
ms=t(lambda: x.sum()); print("read (sum) GB/s", 2*1024**3/ms/1e6)
