"""Forward error of V / tau / R against the oracle on a graded-spectrum input (diagnostic for reading Z24:
V's forward error scales with u * kappa, R's does not)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import inputs, oracle
import paper_2507_00976_b200 as bq

for n, sl in [(512, 1e-10), (512, 1e-4), (512, 1.0)]:
    A, _ = inputs.graded(n, n, n, sigma_last=sl, seed=n)
    A = np.asfortranarray(A)
    o = oracle.bqrrp(A, 64, 80, seed=3)
    Ag, tg, Jg, rk = bq.factor(torch.tensor(np.ascontiguousarray(A.T), device="cuda").t(), 64, 80, seed=3)
    Ag, tg, Jg = Ag.cpu().numpy(), tg.cpu().numpy(), Jg.cpu().numpy()
    l = o.rank
    dR = np.linalg.norm(np.triu(Ag)[:l] - np.triu(o.A)[:l]) / np.linalg.norm(np.triu(o.A)[:l])
    dV = np.linalg.norm(np.tril(Ag, -1) - np.tril(o.A, -1)) / np.linalg.norm(np.tril(o.A, -1))
    # per block column forward error of V
    blk = [float(np.linalg.norm(np.tril(Ag, -1)[:, c:c + 64] - np.tril(o.A, -1)[:, c:c + 64])) for c in range(0, n, 64)]
    print(f"sigma_last {sl:g}: rank {rk}/{l} sameJ {np.array_equal(Jg, o.J)} dR {dR:.2e} dV {dV:.2e} "
          f"dtau {np.max(np.abs(tg - o.tau)):.2e} margin {o.min_margin:.2e} dV per block {['%.0e' % x for x in blk]}")
