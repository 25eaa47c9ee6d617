"""Developer probe: factor + two compressions at config cid, per-level phase times (RSF_PROFILE=1)."""
import sys, time
import torch
sys.path.insert(0, '/root/repo')
from workloads import config, points_for
import paper_1603_08057_b200 as R
cid = int(sys.argv[1]); reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
c = config(cid)
dev = torch.device('cuda:0')
ctx = R.Context(0)
K = R.Kernel(c.family, c.rho, c.sigma2, c.nugget, c.alpha, c.theta)
xy = torch.from_numpy(points_for(c)).to(dev)
for rep in range(reps):
    if rep == reps - 1:
        R.lib.rsf_profile_reset()
    torch.cuda.synchronize(); t = time.time()
    F = R.Factor(ctx, xy, K, c.eps_fact, c.leaf); torch.cuda.synchronize(); tf = time.time() - t
    t = time.time()
    Fi = [] if __import__('os').environ.get('ONLY_SIGMA') == '1' else \
        [R.Factor(ctx, xy, K, c.eps_fact, c.leaf, which=i) for i in range(len(c.theta)) if c.theta[i] in ('rho', 'alpha')]
    torch.cuda.synchronize(); tc = time.time() - t
    info = F.info()
    fl = info.flops_id + info.flops_elim + info.flops_top
    print(f'rep {rep}: factor {tf:.3f}s ({fl/1e12:.2f} TF algorithmic -> {fl/tf/1e12:.2f} TF/s), compressions {tc:.3f}s')
    del F, Fi
prof = R.lib.rsf_profile_dump().decode()
items = sorted([(float(v), k) for k, v in (x.split("=") for x in prof.strip(";").split(";") if "=" in x)], reverse=True) if prof else []
print('PROFILE', ' '.join(f'{k}={v:.3f}' for v, k in items))
if __import__('os').environ.get('RSF_KTRACE') == '1':
    rows = [x.rsplit("=", 1) for x in R.lib.rsf_trace_dump().decode().split(";") if "=" in x]
    rows = sorted(((float(v.split(",")[0]), k, v) for k, v in rows), reverse=True)[:40]
    for sec, k, v in rows:
        print(f"   {sec * 1e3:9.3f} ms  {k}  {v}", flush=True)
