import torch,time
n=367_488_000
d=torch.empty(n,dtype=torch.uint8,device='cuda'); h=torch.empty(n,dtype=torch.uint8).pin_memory()
for chunk in [n, n//20, n//200]:
    torch.cuda.synchronize()
    for rep in range(3):
        t=time.perf_counter()
        for i in range(0,n,chunk): h[i:i+chunk].copy_(d[i:i+chunk],non_blocking=True)
        torch.cuda.synchronize(); dt=time.perf_counter()-t
    print("d2h chunk",chunk,"GB/s",n/dt/1e9)
t=time.perf_counter(); d.copy_(h,non_blocking=True); torch.cuda.synchronize(); print("h2d GB/s",n/(time.perf_counter()-t)/1e9)
