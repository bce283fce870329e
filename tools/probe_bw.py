import torch, json
def t(f, reps=20):
    for _ in range(3): f()
    e0,e1=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
    best=1e9
    for _ in range(3):
        e0.record()
        for _ in range(reps): f()
        e1.record(); torch.cuda.synchronize()
        best=min(best,e0.elapsed_time(e1)/reps)
    return best
n=1<<30
a=torch.empty(n,dtype=torch.float32,device='cuda').normal_()
b=torch.empty_like(a)
r={}
ms=t(lambda: a.sum()); r['sum_f32_4GiB_GBps']=4*n/ms/1e6
ad=a.view(torch.float64)
ms=t(lambda: ad.sum()); r['sum_f64_GBps']=4*n/ms/1e6
ms=t(lambda: b.copy_(a)); r['copy_GBps']=8*n/ms/1e6
ms=t(lambda: b.fill_(1.0)); r['fill_GBps']=4*n/ms/1e6
ms=t(lambda: torch.dot(a,b)); r['dot_f32_GBps']=8*n/ms/1e6
bd=b.view(torch.float64)
ms=t(lambda: torch.dot(ad,bd)); r['dot_f64_GBps']=8*n/ms/1e6
ms=t(lambda: ad.abs().max()) ; r['absmax_f64(2 pass)_ms']=ms
print(json.dumps(r))
