import torch
torch.manual_seed(0)
def t(fn, it=50):
    for _ in range(5): fn()
    torch.cuda.synchronize()
    a,b=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(it): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b)/it*1e3
for (K,N) in [(4096,6144),(4096,4096),(4096,28672),(14336,4096)]:
    W=torch.randn(K,N,device='cuda',dtype=torch.bfloat16)
    for M in (96, 128):
        x=torch.randn(M,K,device='cuda',dtype=torch.bfloat16)
        t1=t(lambda: torch.mm(x,W,out_dtype=torch.float32))
        t2=t(lambda: torch.mm(W.t(),x.t(),out_dtype=torch.float32))
        gb=K*N*2/1e9
        print(f"K={K} N={N} M={M}: x@W {t1:.1f} us ({gb/t1*1e6:.0f} GB/s)  (W^T x^T) {t2:.1f} us ({gb/t2*1e6:.0f} GB/s)")
