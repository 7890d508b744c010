import torch, time
C = torch.empty(93312 * 1600, device="cuda")
for name, fn in (("fill", lambda: C.fill_(1.0)), ("copy", lambda: C.copy_(C.flip(0)) if False else C.mul_(1.0001))):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10): fn()
    b.record(); b.synchronize()
    t = a.elapsed_time(b) / 10 / 1e3
    print(f"{name}: {t*1e3:.3f} ms  {C.numel()*4/t/1e9:.0f} GB/s (write side)")
