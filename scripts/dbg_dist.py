import faulthandler, sys; faulthandler.enable()
sys.path.insert(0, '.')
import numpy as np, torch, synth, paper_1811_05704_b200 as amgb
p,c,v,f = synth.problem("poisson", 32)
multi = amgb.setup_dist(p, c, v, nranks=2, rank=-1, gather_below=500, coarse_enough=100)
print("setup ok", multi.dist_info(), flush=True)
x, it, rel, st = multi.solve(torch.from_numpy(f).cuda(), tol=1e-8, maxiter=200)
print("solve", it, rel, st, flush=True)
