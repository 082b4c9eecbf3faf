"""Write-only HBM bandwidth probes (torch fill_ / memset of a 4 GiB buffer)."""
import torch
dev=torch.device("cuda",0)
def t(fn, nbytes):
    e0,e1=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
    best=1e9
    for k in range(6):
        torch.cuda.synchronize(); e0.record(); fn(k); e1.record(); torch.cuda.synchronize()
        if k: best=min(best,e0.elapsed_time(e1))
    return nbytes/(best/1e3)/1e9
n=4*2**30
b8=torch.empty(n,dtype=torch.uint8,device=dev)
print("u8 fill", t(lambda k: b8.fill_(k+1), n))
print("zero_ (memset)", t(lambda k: b8.zero_(), n))
b64=b8.view(torch.int64)
print("i64 fill", t(lambda k: b64.fill_(k+1), n))
b4=b8.view(torch.float32)
print("f32 fill", t(lambda k: b4.fill_(k+1.0), n))
import ctypes
cudart=ctypes.CDLL("libcudart.so") if False else None
