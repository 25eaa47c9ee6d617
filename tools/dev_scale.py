"""Developer probe: one gp_mle_eval at config cid, size n (z = F^{1/2} w from the CUDA path)."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, '/root/repo')
from workloads import config, points_for, w_for
import paper_1603_08057_b200 as R

cid = int(sys.argv[1]); n = int(sys.argv[2]) if len(sys.argv) > 2 else None
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
c = config(cid)
n = n or c.n
dev = torch.device('cuda:0')
t = time.time()
xy = torch.from_numpy(points_for(c, n)).to(dev)
w = torch.from_numpy(w_for(c, n)).to(dev)
print('inputs', time.time() - t, flush=True)
ctx = R.Context(0)
K = R.Kernel(c.family, c.rho, c.sigma2, c.nugget, c.alpha, c.theta)
t = time.time(); F = R.Factor(ctx, xy, K, c.eps_fact, c.leaf); torch.cuda.synchronize(); tf = time.time() - t
info = F.info()
print(f'factor {tf:.3f}s L={info.levels} top={info.top_size} flops id/elim/top {info.flops_id:.3e} {info.flops_elim:.3e} {info.flops_top:.3e} bytes {info.factor_bytes:.3e}', flush=True)
for l in range(1, info.levels + 1):
    print('  level', l, 'boxes', info.level_boxes[l], 'active', info.level_active[l], 'skel', info.level_skel[l], 'maxI', info.level_maxI[l])
z = F.sample(w)
del F
torch.cuda.synchronize()
free, tot = torch.cuda.mem_get_info(); print('mem free/total GB', free / 1e9, tot / 1e9, flush=True)
for rep in range(reps):
    R.lib.rsf_profile_reset()
    t = time.time()
    r = R.gp_mle_eval(ctx, xy, z, K, c.eps_fact, c.leaf, R.Opts(eps_peel=c.eps_peel, seed=c.seed, probe_block=int(__import__('os').environ.get('PROBE_BLOCK', '512')), peel_f32=int(__import__('os').environ.get('PEEL_F32', '0'))))
    el = time.time() - t
    d = r.diag
    if __import__('os').environ.get('RSF_KTRACE') == '1':
        trr = R.lib.rsf_trace_dump().decode()
        print('   alloc:', ' '.join(x for x in trr.split(';') if x.startswith('alloc') or x.startswith('host-')))
        if rep < reps - 1:
            R.lib.rsf_profile_reset()
    print(f'eval {el:.3f}s ell={r.ell:.10e} grad={r.grad} tree {d.t_tree:.3f} factor {d.t_factor:.3f} compress {d.t_compress:.3f} solve {d.t_solve:.3f} peel {d.t_peel:.3f} launches {d.kernel_launches:.0f}', flush=True)
    for i in range(len(c.theta)):
        p = d.peel[i]
        print('  peel', c.theta[i], 'trace', d.trace[i], 'q', d.q[i], 'cols', list(p.cols)[:p.levels + 1], 'ranks', list(p.rank_max)[:p.levels + 1], 'nL', p.nL, 'cancel', p.cancellation, 'applies', p.applies, 'secs', p.seconds)
free, tot = torch.cuda.mem_get_info(); print('mem free/total GB', free / 1e9, tot / 1e9)
prof = R.lib.rsf_profile_dump().decode()
if prof:
    items = sorted([(float(v), k) for k, v in (x.split('=') for x in prof.strip(';').split(';'))], reverse=True)
    print('PROFILE', ' '.join(f'{k}={v:.3f}' for v, k in items))

tr = R.lib.rsf_trace_dump().decode()
if tr:
    rows = []
    for item in tr.strip(';').split(';'):
        k, v = item.rsplit('=', 1)
        sec, cnt, host = v.split(',')
        rows.append((float(sec), int(cnt), k, float(host)))
    rows.sort(reverse=True)
    tot = sum(r[0] for r in rows)
    print(f'KTRACE total {tot:.3f} s over {sum(r[1] for r in rows)} launches')
    for sec, cnt, k, host in rows[:45]:
        print(f'  {sec:8.3f} s {100*sec/tot:5.1f}% {cnt:7d}  host {host:8.3f} s  {k}')

gl = R.lib.rsf_debug_gemm_log().decode()
if gl:
    rows = []
    for x in gl.strip(';').split(';'):
        k, v = x.rsplit('=', 1)
        sec, fl, cnt, c0, c1, k0, k1, om = v.split(',')
        rows.append((float(sec), float(fl), int(float(cnt)), k, c0, c1, k0, k1, om))
    rows.sort(reverse=True)
    tot = sum(r[0] for r in rows)
    print(f'GEMMLOG total {tot:.3f} s over {sum(r[2] for r in rows)} launches, {sum(r[1] for r in rows)/tot/1e12:.2f} TF/s')
    for sec, fl, cnt, k, c0, c1, k0, k1, om in rows[:400]:
        print(f'  {sec:8.3f} s {100*sec/tot:5.1f}% {fl/max(sec,1e-12)/1e12:6.2f} TF/s n={cnt:6d} ctas {c0}-{c1} K {k0}-{k1} longest#{om}  {k}')
