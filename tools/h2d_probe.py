import torch, time
x = torch.empty(652_000_000, dtype=torch.uint8).pin_memory()
y = torch.empty_like(x, device="cuda")
s = torch.cuda.Stream()
for chunks in (1, 16, 96):
    n = x.numel() // chunks
    for rep in range(3):
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(s)
        with torch.cuda.stream(s):
            for c in range(chunks):
                y[c*n:(c+1)*n].copy_(x[c*n:(c+1)*n], non_blocking=True)
        e1.record(s); e1.synchronize()
        ms = e0.elapsed_time(e1)
    print(chunks, "chunks", round(ms,2), "ms", round(x.numel()/ms/1e6,1), "GB/s")
# duplex: H2D and D2H concurrently
z = torch.empty(104_000_000, dtype=torch.uint8, device="cuda"); zh = torch.empty(104_000_000, dtype=torch.uint8).pin_memory()
s2 = torch.cuda.Stream()
torch.cuda.synchronize(); t0=time.perf_counter()
with torch.cuda.stream(s): y.copy_(x, non_blocking=True)
with torch.cuda.stream(s2): zh.copy_(z, non_blocking=True)
torch.cuda.synchronize(); print("duplex", round((time.perf_counter()-t0)*1e3,2), "ms")
