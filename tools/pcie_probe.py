import torch, time
dev=torch.device("cuda",0)
for mb in (1,2,4,8,16):
    n=mb*(1<<20)//8
    d=torch.empty(n,dtype=torch.float64,device=dev)
    hs=[torch.empty(n,dtype=torch.float64).pin_memory() for _ in range(4)]
    ss=[torch.cuda.Stream() for _ in range(4)]
    for mode in ("one stream","4 streams"):
        torch.cuda.synchronize(); 
        reps=400
        t0=time.perf_counter()
        for i in range(reps):
            s=ss[i%4] if mode=="4 streams" else ss[0]
            with torch.cuda.stream(s): hs[i%4].copy_(d,non_blocking=True)
        torch.cuda.synchronize(); dt=time.perf_counter()-t0
        print(f"D2H {mb} MB {mode}: {mb*1.048576*reps/dt/1e3:.1f} GB/s")
    # graph of copies
    g=torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for i in range(8): hs[i%4].copy_(d,non_blocking=True)
    g.replay(); torch.cuda.synchronize()
    t0=time.perf_counter()
    for _ in range(50): g.replay()
    torch.cuda.synchronize(); dt=time.perf_counter()-t0
    print(f"D2H {mb} MB graph x8: {mb*1.048576*8*50/dt/1e3:.1f} GB/s")
