import time, torch
dev=torch.device("cuda",0)
gat=torch.cuda.Stream()
shape=(100000,1024)
keep=[]
warm=[torch.empty(shape,device=dev) for _ in range(4)]; del warm
ts=[]
for i in range(300):
    t=time.perf_counter()
    b=torch.empty(shape,device=dev)
    ts.append(time.perf_counter()-t)
    b.record_stream(gat)
    with torch.cuda.stream(gat):
        b[:1000].fill_(1.0)
    keep.append(b)
    if len(keep)>2: keep.pop(0)
import numpy as np
ts=np.array(ts)*1e6
print("alloc us median %.1f mean %.1f p90 %.1f max %.1f"%(np.median(ts),ts.mean(),np.percentile(ts,90),ts.max()))
print({k:v for k,v in torch.cuda.memory_stats().items() if k in ("num_device_alloc","num_device_free","num_alloc_retries")})
