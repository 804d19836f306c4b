import torch, time, numpy as np
dev=torch.device("cuda",0)
for mb in (1,2,4,8,16,32,64,128):
    n=mb*1024*1024//4
    h=torch.empty(n).pin_memory(); d=torch.empty(n,device=dev)
    for direction in ("h2d","d2h"):
        ts=[]
        for _ in range(7):
            torch.cuda.synchronize(); t0=time.perf_counter()
            if direction=="h2d": d.copy_(h,non_blocking=True)
            else: h.copy_(d,non_blocking=True)
            torch.cuda.synchronize(); ts.append(time.perf_counter()-t0)
        t=np.median(ts); print(f"{mb:4d} MB {direction}: {1e3*t:.3f} ms {mb/1024/t:.1f} GB/s")
