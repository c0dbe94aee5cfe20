import sys, numpy as np, torch
sys.path.insert(0, '.')
import oracle, synth
from paper_2407_20692_b200 import Context
def run(wa, ha, wb, hb, alphas, boundary, seed, verbose=True):
    dims = (wa, ha, wb, hb)
    G = synth.random_gamma(wa * ha, wb * hb, seed=seed)
    ctx = Context((0, 0, wa, ha), (0, 0, wb, hb), 1)
    g = torch.from_numpy(np.ascontiguousarray(G, dtype=np.float32)).cuda()
    planes = ctx.new_planes(len(alphas))
    ctx.refocus(alphas, g, planes, boundary=boundary)
    torch.cuda.synchronize()
    R = planes.cpu().numpy().astype(np.float64)
    Ro = oracle.refocus(G, dims, alphas, boundary=boundary)
    M = oracle.refocus(np.abs(G.astype(np.float64)), dims, alphas, boundary=boundary)
    bad = ~(np.abs(R - Ro) <= 1e-6 * M + 1e-30)
    ctx.close()
    if verbose or bad.any():
        print(dims, alphas, boundary, seed, 'bad', int(bad.sum()), 'of', bad.size, 'shape', R.shape)
        for idx in list(zip(*np.nonzero(bad)))[:8]:
            print('   ', idx, R[idx], Ro[idx], M[idx])
    return bad.any()
run(3, 18, 3, 4, [2.00001], 0, 189)
run(3, 18, 3, 4, [2.0], 0, 189)
run(3, 18, 3, 4, [2.00001], 1, 189)
run(4, 18, 3, 4, [2.00001], 0, 189)
run(3, 18, 4, 4, [2.00001], 0, 189)
rng = np.random.default_rng(0)
nb = 0
for k in range(60):
    wa, ha, wb, hb = int(rng.integers(2, 41)), int(rng.integers(2, 31)), int(rng.integers(1, 21)), int(rng.integers(1, 13))
    al = [float(a) for a in rng.uniform(0.3, 2.5, size=int(rng.integers(1, 7)))]
    nb += run(wa, ha, wb, hb, al, int(rng.integers(0, 2)), int(rng.integers(0, 2**31 - 1)), verbose=False)
for a in [1.99999, 2.00001, 2.0001, 2.01, 2.3, 2.5]:
    for wa in [2, 3, 5, 8]:
        nb += run(wa, 18, 3, 4, [a], 0, 7, verbose=False)
print('random bad', nb)
