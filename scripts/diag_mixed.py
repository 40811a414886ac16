import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth, paper_1811_05704_b200 as amgb
for n in (32, 64, 128):
    p, c, v, f = synth.poisson3d(n)
    hm = amgb.setup(p, c, v, precision="mixed"); hd = amgb.setup(p, c, v)
    r = torch.from_numpy(synth.random_vector(len(f))).cuda()
    zm = hm.precond(r).cpu().numpy(); zd = hd.precond(r).cpu().numpy()
    fd = torch.from_numpy(f).cuda()
    xm, im, rm, _ = hm.solve(fd, tol=1e-8); xd, idd, rd, _ = hd.solve(fd, tol=1e-8)
    xm = xm.cpu().numpy(); xd = xd.cpu().numpy()
    print(n, 'precond rel diff %.2e' % (np.linalg.norm(zm - zd) / np.linalg.norm(zd)), 'iters', im, idd,
          'x rel diff %.2e' % (np.linalg.norm(xm - xd) / np.linalg.norm(xd)), 'res', rm, rd,
          'bytes/vc', hm.level_info(0)['alg_bytes_vcycle'], hd.level_info(0)['alg_bytes_vcycle'], flush=True)
