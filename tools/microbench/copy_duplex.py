import torch, time
a = torch.empty(48<<20, dtype=torch.uint8).pin_memory(); b = torch.empty(58<<20, dtype=torch.uint8).pin_memory()
da = torch.empty(48<<20, dtype=torch.uint8, device='cuda'); db = torch.empty(58<<20, dtype=torch.uint8, device='cuda')
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for rep in range(3):
    torch.cuda.synchronize(); t=time.perf_counter()
    with torch.cuda.stream(s1): da.copy_(a, non_blocking=True)
    torch.cuda.synchronize(); t1=time.perf_counter()
    with torch.cuda.stream(s2): b.copy_(db, non_blocking=True)
    torch.cuda.synchronize(); t2=time.perf_counter()
    with torch.cuda.stream(s1): da.copy_(a, non_blocking=True)
    with torch.cuda.stream(s2): b.copy_(db, non_blocking=True)
    torch.cuda.synchronize(); t3=time.perf_counter()
    print(f"h2d 48MB {1e3*(t1-t):.3f} ms ({48*1.048576/(t1-t)/1e3:.1f} GB/s)  d2h 58MB {1e3*(t2-t1):.3f} ms  both {1e3*(t3-t2):.3f} ms")
