"""PCIe bound of the headline e2e: pinned H2D of X (6.5 MB fp16), D2H of Y (12.8 MB fp32),
each alone and both concurrently (two streams), CUDA-event timed (debug aid)."""
import torch

x = torch.empty(6496256 // 2, dtype=torch.float16).pin_memory()
y = torch.empty(12845056 // 4, dtype=torch.float32).pin_memory()
dx = torch.empty_like(x, device="cuda")
dy = torch.empty_like(y, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def t(fn, n=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e3


def both():
    with torch.cuda.stream(s1):
        dx.copy_(x, non_blocking=True)
    with torch.cuda.stream(s2):
        y.copy_(dy, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)


print("H2D 6.5 MB us", round(t(lambda: dx.copy_(x, non_blocking=True)), 1))
print("D2H 12.8 MB us", round(t(lambda: y.copy_(dy, non_blocking=True)), 1))
print("both concurrent us", round(t(both), 1))
