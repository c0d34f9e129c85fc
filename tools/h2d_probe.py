"""Pinned host -> device copy bandwidth (one copy, 2/4 concurrent streams, 8 MB chunks).
Usage: python tools/h2d_probe.py"""
import time, torch
N = 128*512*512
h = torch.rand(N).pin_memory()
d = torch.empty(N, device="cuda")
def bw(fn, reps=5):
    fn(); torch.cuda.synchronize(); t=time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize(); return reps*N*4/(time.perf_counter()-t)/1e9
print("single", bw(lambda: d.copy_(h, non_blocking=True)))
streams=[torch.cuda.Stream() for _ in range(4)]
def multi(k):
    def f():
        n=N//k
        for i in range(k):
            with torch.cuda.stream(streams[i]):
                d[i*n:(i+1)*n].copy_(h[i*n:(i+1)*n], non_blocking=True)
        for s in streams[:k]: torch.cuda.current_stream().wait_stream(s)
    return f
print("2 streams", bw(multi(2))); print("4 streams", bw(multi(4)))
# zero-copy: kernel reads pinned host memory (UVA) -- torch elementwise on a host tensor isn't allowed; use cupy-free trick: torch can't. skip
# chunked 8MB copies on one stream
def chunked():
    n=2*1024*1024
    for i in range(0,N,n): d[i:i+n].copy_(h[i:i+n], non_blocking=True)
print("chunked 8MB", bw(chunked))
