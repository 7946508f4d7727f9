"""Does a device-to-host copy on one stream overlap kernels on another?
(probe for the pipelined host entry). Prints ms for copy alone, compute alone, both."""
import torch
dev = torch.device("cuda", 0)
n = 4 << 30
src = torch.empty(n, dtype=torch.uint8, device=dev)
dst = torch.empty(n, dtype=torch.uint8, pin_memory=True)
a = torch.randn(8192, 8192, device=dev)
s_cp = torch.cuda.Stream()
s_k = torch.cuda.Stream()


def timed(fn):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    fn()
    torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)


def copy():
    with torch.cuda.stream(s_cp):
        dst.copy_(src, non_blocking=True)


def comp():
    with torch.cuda.stream(s_k):
        for _ in range(40):
            torch.mm(a, a)


for _ in range(2):
    tc, tk = timed(copy), timed(comp)
    tb = timed(lambda: (copy(), comp()))
    print(f"copy {tc:.1f} ms ({n / tc / 1e6:.1f} GB/s), compute {tk:.1f} ms, both {tb:.1f} ms")
