import torch
x = torch.empty(1 << 28, dtype=torch.float32, device="cuda")
y = torch.empty_like(x)
x.normal_()
def t(f, nbytes, reps=20):
    for _ in range(3): f()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(reps):
        e0.record(); f(); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return nbytes / best / 1e6
print("write (fill_)", t(lambda: y.fill_(1.0), 4 << 28))
print("write (zero_)", t(lambda: y.zero_(), 4 << 28))
print("copy", t(lambda: y.copy_(x), 8 << 28))
print("read (amax)", t(lambda: x.abs().max(), 4 << 28 + 0))
