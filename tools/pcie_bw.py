import torch, time
dev=torch.device("cuda",0)
for mb in (256, 1536):
    n=mb*1024*1024
    h=torch.empty(n,dtype=torch.uint8).pin_memory(); d=torch.empty(n,dtype=torch.uint8,device=dev)
    for _ in range(2): d.copy_(h,non_blocking=True); h.copy_(d,non_blocking=True)
    torch.cuda.synchronize()
    s,e=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
    s.record(); d.copy_(h,non_blocking=True); e.record(); torch.cuda.synchronize(); t1=s.elapsed_time(e)
    s.record(); h.copy_(d,non_blocking=True); e.record(); torch.cuda.synchronize(); t2=s.elapsed_time(e)
    print(f"{mb} MiB: H2D {n/t1/1e6:.1f} GB/s  D2H {n/t2/1e6:.1f} GB/s")
