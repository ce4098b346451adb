import sys, time, torch, os
sys.path.insert(0, '/root/repo')
from paper_2009_10863_b200 import InitialGuess, ig_form_guess_host, ig_update_host
from workloads.gen import manufactured_step_slab
n=128; N=n**3; M=8
pool=[manufactured_step_slab(n,n,0,1,k,device='cuda') for k in range(20)]
hp=InitialGuess(N,'proj_qr',M); he=InitialGuess(N,'extrap_ls',M,3)
x0p=torch.zeros(N,dtype=torch.float64,device='cuda'); x0e=torch.zeros_like(x0p)
for k in range(12):
    b,x,Ax=pool[k]; hp.form_guess(b,x0p); hp.update(x,Ax); he.form_guess(None,x0e); he.update(x)
torch.cuda.synchronize()
for PH in (4, 9, 9, 4):
    host=[tuple(t.cpu().pin_memory() for t in pool[j]) for j in range(PH)]
    a=torch.zeros(N,dtype=torch.float64).pin_memory(); c=torch.zeros(N,dtype=torch.float64).pin_memory()
    for KE in (20,):
        t0=time.perf_counter()
        for j in range(KE):
            b,x,Ax=host[j%PH]
            ig_form_guess_host(hp.h,b,a); ig_update_host(hp.h,x,Ax); ig_form_guess_host(he.h,None,c); ig_update_host(he.h,x,None)
        torch.cuda.synchronize(); dt=(time.perf_counter()-t0)/KE
        print(PH, KE, f"{dt*1e3:.2f} ms/step", hp.stats()['admitted'])
