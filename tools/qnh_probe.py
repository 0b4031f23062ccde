import sys, time, os
sys.path.insert(0, '/root/repo')
import torch, numpy as np, workloads as W, paper_2305_11645_b200 as rq
prob = W.make_config(sys.argv[1])
pl = rq.Plan.from_problem(prob)
print([ (L['w'], L['coarse'], L['absorbed'], L['fft']) for L in pl.levels()])
A_pin = torch.from_numpy(prob.A.copy()).pin_memory(); Ah = A_pin.numpy()
for _ in range(3): pl.qn_host(Ah, prob.f, prob.fparam)
torch.cuda.synchronize()
ts=[]
for _ in range(20):
    t=time.perf_counter(); pl.qn_host(Ah, prob.f, prob.fparam); ts.append(time.perf_counter()-t)
print("RES qn_host ms", np.median(ts)*1e3, min(ts)*1e3)
A = torch.from_numpy(prob.A).cuda(); out=torch.empty(1,dtype=torch.float64,device='cuda')
for _ in range(3): pl.qn_sum(A, prob.f, prob.fparam, out=out)
torch.cuda.synchronize(); ts=[]
for _ in range(20):
    t=time.perf_counter(); pl.qn_sum(A, prob.f, prob.fparam, out=out); torch.cuda.synchronize(); ts.append(time.perf_counter()-t)
print("RES qn_sum+sync ms", np.median(ts)*1e3, min(ts)*1e3)
