import os, sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
import oracle, workloads as W, paper_2305_11645_b200 as rq
def run(prob, env):
    for k, v in env.items(): os.environ[k] = v
    p = rq.Plan.from_problem(prob)
    from torch.profiler import profile, ProfilerActivity
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        Y, fs = p.xa(torch.from_numpy(prob.A).cuda(), prob.f, prob.fparam); torch.cuda.synchronize()
    print(sorted(set(e.name[:40] for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA)))
    Yg = Y.cpu().numpy()
    Xs = oracle.points_rows(prob, np.arange(prob.N)); Yo = oracle.product(Xs, prob.A)
    err = np.abs(Yg - Yo).max(axis=1)
    bad = np.nonzero(err > 1e-9)[0]
    print(env, [L['absorbed'] for L in p.levels()], 'bad rows', len(bad), bad[:10], err.max())
for mp in (W.MAP_INVNORM, W.MAP_UNIT):
  prob = W.make_random(201, 2, 12, 150, 48, shifted=True, mapping=mp, f=W.F_EXP_MEAN)
  for env in [dict(RQMC_ABSORB='0', RQMC_GEMM_LAT='0'), dict(RQMC_ABSORB='0', RQMC_GEMM_LAT='1'), dict(RQMC_ABSORB='', RQMC_GEMM_LAT='')]:
    run(prob, env)
